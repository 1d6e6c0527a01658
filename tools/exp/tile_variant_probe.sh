#!/bin/bash
for lib in "" tools/exp/variants/liblpt1.so tools/exp/variants/liblpt3.so tools/exp/variants/liblpt4.so; do
  if [ -n "$lib" ]; then export MPMM_LIB_PATH=$lib; else unset MPMM_LIB_PATH; fi
  python tools/exp/tile_variant_probe.py
done
