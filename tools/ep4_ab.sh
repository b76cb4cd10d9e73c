#!/bin/bash
# EP=4 A/B of opt-in variants against the default: timelines, twice. Usage: bash tools/ep4_ab.sh VAR=VAL ...
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
VARS=${*:-B2_EP_OVERLAP_PULL=1}
for i in 1 2; do
  for v in NONE $VARS; do
    echo "== $v"
    env $( [ $v = NONE ] || echo $v ) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/timeline.py --graph 2>&1 | grep -E "event-timed|combine_slots|pull_sum_kernel<__nv|gather_pull" | head -5
  done
done
