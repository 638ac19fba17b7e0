#!/bin/bash
# Profile one short bench run on the GPU box (run under gpurun, from the repo root).
#   tools/profile.sh TAG [KERNEL_REGEX] [SKIP]
# 1) plain run (must exit 0), 2) ncu launch list (per-launch device time),
# 3) ncu --set full of one launch of the top kernel.  Outputs in gpurun_out/.
TAG=${1:-run}
KREGEX=${2:-k_update}
SKIP=${3:-21}
ARGS=${PROFILE_ARGS:-"--batch 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 1"}
mkdir -p gpurun_out
timeout 600 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $SKIP -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
