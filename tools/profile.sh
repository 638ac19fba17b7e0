#!/bin/bash
# Profile one short bench run on the GPU box (run under gpurun, from the repo root).
#   tools/profile.sh TAG [KERNEL_REGEX:SKIP ...]
# 1) plain run (must exit 0), 2) ncu launch list (per-launch device time),
# 3) one ncu --set full capture per KERNEL_REGEX:SKIP pair (default: the level-0
#    t=1 message update and the second JBU launch).  Outputs in gpurun_out/.
TAG=${1:-run}
shift
CAPS=${@:-"k_update_fast:21 k_jbu_fast:1"}
ARGS=${PROFILE_ARGS:-"--batch 256 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pairs 512"}
mkdir -p gpurun_out
timeout 600 python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
for cap in $CAPS; do
    K=${cap%%:*}
    S=${cap##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
        -o gpurun_out/prof_${TAG}_$K python bench.py $ARGS > gpurun_out/ncu_full_${TAG}_$K.log 2>&1
    echo "full $K rc=$?"
done
