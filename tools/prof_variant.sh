#!/bin/bash
# usage: tools/prof_variant.sh lib.so out_name  (runs prof_run with MHFD_LIB=lib and ncu on k_band)
export MHFD_LIB=$(realpath $1)
python tools/prof_run.py --batch 2 > gpurun_out/prof_plain_$2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_band -s 1 -c 1 -o gpurun_out/$2 python tools/prof_run.py --batch 2 > gpurun_out/prof_ncu_$2.log 2>&1
