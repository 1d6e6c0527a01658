#!/bin/bash
# TILE_32 (n_min 32) register-tile variants: -DMPMM_DD32_CFG=2,4,5,6
for lib in "" tools/exp/vl/libdd32_2.so tools/exp/vl/libdd32_4.so tools/exp/vl/libdd32_5.so tools/exp/vl/libdd32_6.so; do
  if [ -n "$lib" ]; then export MPMM_LIB_PATH=$lib; else unset MPMM_LIB_PATH; fi
  python tools/exp/tile_variant_probe.py 2>&1 | grep "n_min=32"
done
