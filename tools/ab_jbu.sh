#!/bin/bash
# A/B of JBU builds on one box (run under gpurun): tools/ab_jbu.sh TAG variant...
# ("base" = the in-tree libvsbp.so); two interleaved rounds; JSON lines in gpurun_out/ab_TAG.log
TAG=$1; shift
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
  if [ $v = base ]; then L=; else L=$PWD/exp/libvsbp_$v.so; fi
  VSBP_LIB=$L timeout 300 python tools/time_jbu.py --tag $v >> gpurun_out/ab_$TAG.log 2>&1
done; done
cat gpurun_out/ab_$TAG.log
