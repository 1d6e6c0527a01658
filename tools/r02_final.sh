#!/bin/bash
# Round-2 validation of the current tree on one B200: smoke, the GPU test
# suite, the bench (both arms) and the bench's ncu launch list.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu.log
python bench.py > gpurun_out/r02_bench.jsonl 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r02_bench_reference.jsonl 2> gpurun_out/r02_bench_reference.err; echo "ref rc=$?"
# the launch list of the same command at the block size the bench's predictor
# chose (under ncu every launch is serialised and cold, which would skew the
# predictor's slice timings and with them the kernel the step launches)
NMIN=$(python -c "import json; print([json.loads(l) for l in open('gpurun_out/r02_bench.jsonl') if l.startswith('{')][-1]['block_size']['n_min'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 \
  --nmin $NMIN --no-cpu-baseline --no-extras > gpurun_out/r02_ncu_bench.log 2>&1; echo "ncu rc=$? (n_min $NMIN)"
