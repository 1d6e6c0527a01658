#!/bin/bash
# BASELINE configs[4]: the tuner on the seed-1 inputs, sizes 512..8192,
# GPU counts 1/2/4/8 (G > 1: shard product measured + broadcast model),
# Strassen cutoffs tuned; warm measurements.
set -u
python -m paper_1710_01839_b200 tune --prec dd --dims 512,1024,2048,4096,8192 \
  --nmin 16,32,64,128,256 --threads 1 --gpus 1,2,4,8 --cutoffs 32,64,128,256,512,1024,2048 \
  --inputs seeded --seed 1 --warmup 1 --repeats 2 --agg min \
  --out gpurun_out/r02_cfg4_dd.tbl > gpurun_out/r02_tune_dd.log 2>&1
echo "dd rc=$?"
python -m paper_1710_01839_b200 tune --prec qd --dims 512,1024,2048,4096,8192 \
  --nmin 16,64,256 --threads 1 --gpus 1,2,4,8 --cutoffs 32,64,128,256,1024 \
  --inputs seeded --seed 1 --warmup 0 --repeats 1 --agg min \
  --out gpurun_out/r02_cfg4_qd.tbl > gpurun_out/r02_tune_qd.log 2>&1
echo "qd rc=$?"
for p in dd qd; do
  python -m paper_1710_01839_b200 report --in gpurun_out/r02_cfg4_$p.tbl --format winners
done
