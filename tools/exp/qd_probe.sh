#!/bin/bash
# QD kernel variants (tools/exp/vl/libqd_*.so) through tools/exp/qd_time.py
for lib in ${@:-dense}; do MPMM_LIB_PATH=tools/exp/vl/libqd_$lib.so python tools/exp/qd_time.py 2>&1 | grep -E "n=1024|n=2048|n=512 n_min=64"; done
