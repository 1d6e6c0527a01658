python bench.py > gpurun_out/s2_bench.jsonl 2> gpurun_out/s2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_tensor_dd_launches.csv python tools/prof_tensor.py dd 1024 > gpurun_out/s2_pt_dd.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_tensor_qd_launches.csv python tools/prof_tensor.py qd 1024 > gpurun_out/s2_pt_qd.log 2>&1
python tools/prof_tensor.py dd 1024 >> gpurun_out/s2_pt_dd.log 2>&1
python tools/prof_tensor.py qd 1024 >> gpurun_out/s2_pt_qd.log 2>&1
python tools/prof_tensor.py dd 2048 >> gpurun_out/s2_pt_dd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"combine|residues|scan" -c 6 -o gpurun_out/s2_tensor python tools/prof_tensor.py dd 1024 > gpurun_out/s2_ncu_tensor.log 2>&1
ncu -i gpurun_out/s2_tensor.ncu-rep --page raw --csv > gpurun_out/s2_tensor_raw.csv 2>/dev/null
