#!/bin/bash
# EP=2 A/B of the dispatch-overlap variants: parity tests (unless SKIPTEST) + timelines.
# Usage (gpurun --gpus 2): TAG=sNN bash tools/ep2_fused_check.sh [ENVVAR ...]
set -u
OUT=gpurun_out/${TAG:-ep2ab}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
[ -n "${SKIPTEST:-}" ] || { timeout 900 python -m pytest tests/test_gpu_ep.py -x -q -k "ep_matches and 2-" > $OUT/eptests.log 2>&1; echo "ep tests rc=$?"; tail -3 $OUT/eptests.log; }
VARS=${*:-B2_EP_OVERLAP_PULL}
for i in 1 2; do
  for v in NONE $VARS; do
    echo "== $v"
    env $( [ $v = NONE ] || echo $v=1 ) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/timeline.py --graph 2>&1 | grep -E "event-timed|grouped_gemm|gather_pull|pull_rows|out_reduction" | head -6
  done
done
