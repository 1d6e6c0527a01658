set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1
python bench.py > gpurun_out/r01i_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01i_bench_ref.log 2>&1
MPMM_HOST_STREAMED=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01i_launches_bench.csv python bench.py --steps 3 --warmup 3 --nmin 32 > gpurun_out/r01i_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tiled -c 1 -o gpurun_out/r01i_dd_t32 python tools/prof_kernels.py --prec dd --n 1024 --nmin 32 --reps 2 > gpurun_out/r01i_ncu_dd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tiled -c 1 -o gpurun_out/r01i_qd_t16 python tools/prof_kernels.py --prec qd --n 1024 --nmin 16 --reps 1 > gpurun_out/r01i_ncu_qd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"combine_mma|residues_rows|residue_gemm" -c 3 -o gpurun_out/r01i_tensor python tools/prof_tensor.py dd 1024 > gpurun_out/r01i_ncu_tensor.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i_tensor_dd_launches.csv python tools/prof_tensor.py dd 1024 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i_tensor_qd_launches.csv python tools/prof_tensor.py qd 1024 > /dev/null 2>&1
for f in r01i_dd_t32 r01i_qd_t16 r01i_tensor; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null; done
python -m pytest tests -m gpu -q > gpurun_out/r01i_pytest_gpu.log 2>&1
python tools/e2e_probe.py > gpurun_out/r01i_e2e_probe.log 2>&1
for n in 1024 2048 4096 8192; do python tools/prof_tensor.py dd $n; done > gpurun_out/r01i_tensor_times.log 2>&1
for n in 1024 2048 4096; do python tools/prof_tensor.py qd $n; done >> gpurun_out/r01i_tensor_times.log 2>&1
tail -2 gpurun_out/r01i_pytest_gpu.log
