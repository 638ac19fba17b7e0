#!/bin/bash
# End-of-round evidence (run under gpurun from the repo root):
#   tools/final_round.sh TAG
# 1) all GPU tests, 2) smoke(), 3) the default bench line (N=1, cpu_baseline, e2e),
# 4) the reference (oracle) arm, 5) f-row timings, 6) the ncu launch list of the
# bench command and one --set full capture each of the two-iteration and final
# (last iteration + WTA) level-0 updates, the JBU and the compaction write.  Every step runs without ncu
# first.  Outputs in gpurun_out/.
TAG=${1:-final}
mkdir -p gpurun_out
python -c "from paper_1902_09733_b200 import build as B; B.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
[ -n "$SKIP_ROWS" ] || { timeout 900 python tools/bench_rows.py --out gpurun_out/rows_$TAG.json > /dev/null 2> gpurun_out/rows_$TAG.err; echo "rows rc=$?"; }
ARGS="--batch 256 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pairs 512"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
# k_update_pair launches per step: levels 2 and 1 (u16: MODE 2, MODE 0 each), then level 0 (MODE 2,
# MODE 0, FIN = the last iteration + both WTAs)
for cap in ${CAPS:-k_update_pair:5 k_update_pair:6 k_jbu_vec:1 k_compact_write:1}; do
    K=${cap%%:*}; S=${cap##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
        -o gpurun_out/prof_${TAG}_${K}_s$S python bench.py $ARGS > gpurun_out/ncu_full_${TAG}_${K}_s$S.log 2>&1
    echo "full $K (skip $S) rc=$?"
done
