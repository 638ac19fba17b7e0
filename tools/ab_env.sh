#!/bin/bash
# A/B of whole bench steps under environment settings, alternating, N rounds:
#   tools/ab_env.sh N "VSBP_PAIR_MINPX=50000" "VSBP_PAIR_BAND=32" ...  -> gpurun_out/ab_env.log
# (the first variant of every round is the default environment)
N=$1; shift
mkdir -p gpurun_out
for r in $(seq $N); do
  for v in default "$@"; do
    if [ "$v" = default ]; then E=""; else E="$v"; fi
    env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['us_per_launch'],1))" >> gpurun_out/ab_env.log
  done
done
