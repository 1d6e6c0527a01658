#!/bin/bash
# End-of-session validation: smoke, GPU tests, bench (both arms), e2e probe.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01l_smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/r01l_pytest_gpu.log 2>&1
python bench.py > gpurun_out/r01l_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01l_bench_ref.log 2>&1
python tools/e2e_probe.py > gpurun_out/r01l_e2e_probe.log 2>&1
tail -2 gpurun_out/r01l_pytest_gpu.log
