#!/bin/bash
# One GPU check round (run under gpurun from the repo root):
#   tools/gpu_round.sh TAG [pytest-k-expr]
# rebuilds libvsbp.so if stale, runs the GPU tests, a bench line, the ncu launch
# list (time + DRAM bytes per launch) and one --set full capture of the JBU and
# cost kernels.  Outputs in gpurun_out/.
TAG=${1:-run}
K=${2:-}
mkdir -p gpurun_out
python -c "from paper_1902_09733_b200 import build as B; B.build()" || exit 1
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
fi
tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
ARGS="--batch 16 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
if [ -n "$FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$FULL" -s ${FULL_SKIP:-2} -c ${FULL_COUNT:-2} \
      -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
fi
