#!/bin/bash
# One GPU round trip of measurement evidence (outputs under gpurun_out/, summarised into profiles/ here):
#   plain runs first (each ncu pass only after its command exited 0 without ncu), then
#   (1) per-kernel metrics over the launches of tools/timeline.py 26 (3 H steps: 2 warm-up + 1),
#   (2) the bench line, (3) the launch list of the bench command itself (device time per launch),
#   (4) with FULL=<kernel regex>, one `--set full` capture (3 launches) of those kernels.
set -o pipefail
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-prof}
python tools/timeline.py 26 > gpurun_out/${TAG}_plain_timeline.txt 2>&1 || { echo "plain timeline failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --page raw --log-file gpurun_out/${TAG}_metrics.csv python tools/timeline.py 26 > gpurun_out/${TAG}_ncu1.log 2>&1
echo "metrics rc=$?"
python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || { echo "bench failed"; tail -5 gpurun_out/${TAG}_bench.err; exit 1; }
cat gpurun_out/${TAG}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_ncu2.log 2>&1
echo "launch list rc=$?"
if [ -n "$FULL" ]; then   # the --set full capture is large: run it in its own call (gpurun copies back <= 64 MiB)
ncu --set full --clock-control none --import-source on -k regex:"$FULL" -c 3 \
    -o gpurun_out/${TAG}_full python tools/timeline.py 26 > gpurun_out/${TAG}_ncu3.log 2>&1
echo "full rc=$?"
fi
