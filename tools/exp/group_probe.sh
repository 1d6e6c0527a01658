#!/bin/bash
# tile-raster group size: time and DRAM reads of the 8192^3 DD kernel
for lib in "" tools/exp/variants/libg4.so tools/exp/variants/libg32.so tools/exp/variants/libg64.so; do
  if [ -n "$lib" ]; then export MPMM_LIB_PATH=$lib; else unset MPMM_LIB_PATH; fi
  python tools/exp/group_probe.py
  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --kernel-name-base demangled \
      -k regex:"gemm_tiled<mpmm::DDOps" -s 1 -c 1 python tools/prof_kernel.py dd 8192 32 2>&1 \
      | grep -E "dram__bytes_read|gpu__time_duration" | sed "s|^|  ${lib:-g16} |"
done
