#!/bin/bash
# A/B of whole bench steps on one box: alternating runs of the in-tree libvsbp.so and
# the variants named on the command line (exp/libvsbp_NAME.so), N rounds each.
#   tools/ab_bench.sh N NAME...   -> gpurun_out/ab.log, one line per run
N=$1; shift
mkdir -p gpurun_out
for r in $(seq $N); do
  for v in in-tree "$@"; do
    if [ "$v" = in-tree ]; then L=""; else L="exp/libvsbp_$v.so"; fi
    VSBP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['us_per_launch'],1))" >> gpurun_out/ab.log
  done
done
