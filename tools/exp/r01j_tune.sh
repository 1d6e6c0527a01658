#!/bin/bash
# cfg4: the tuner with the exact-mode candidate, warm measurements
python -m paper_1710_01839_b200 tune --prec dd --dims 512,1024,2048,4096,8192 --nmin 16,32,64,128,256 --threads 1 --cutoffs 256,512,1024,2048 --exact-mode --warmup 1 --repeats 3 --agg min --out gpurun_out/r01j_cfg4_dd.tbl > gpurun_out/r01j_tune_dd.log 2>&1
python -m paper_1710_01839_b200 tune --prec qd --dims 512,1024,2048,4096 --nmin 16,32,64,128,256 --threads 1 --cutoffs 256,512,1024,2048 --exact-mode --warmup 1 --repeats 2 --agg min --out gpurun_out/r01j_cfg4_qd.tbl > gpurun_out/r01j_tune_qd.log 2>&1
for p in dd qd; do python -m paper_1710_01839_b200 report --in gpurun_out/r01j_cfg4_$p.tbl --format winners; done
