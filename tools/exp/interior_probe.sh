#!/bin/bash
# Interior-path variants of the DD blocked kernels (gemm.cuh gemm_tile_interior):
# time per block size and a hash of the 1024^3 result (must agree bit for bit).
export MPMM_PROBE_NMIN=${MPMM_PROBE_NMIN:-32,64,128,256}
for lib in ${@:-off u2 u4 u8 u16}; do
  MPMM_LIB_PATH=tools/exp/vl/libint_$lib.so python tools/exp/tile_variant_probe.py 2>&1 | grep -v Warning
done
