#!/bin/bash
# One GPU round trip: parity tests, smoke, bench (H).  Outputs under gpurun_out/.
set -o pipefail
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-run}
timeout 900 python -m pytest tests/ -m gpu -q -x --tb=short > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
