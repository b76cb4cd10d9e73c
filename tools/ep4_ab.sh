#!/bin/bash
# EP=4 A/B of an opt-in variant (env var set to 1) against the default: timelines, twice.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
VARS=${*:-B2_EP_OVERLAP_PULL}
for i in 1 2; do
  for v in NONE $VARS; do
    echo "== $v"
    env $( [ $v = NONE ] || echo $v=1 ) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/timeline.py --graph 2>&1 | grep -E "event-timed|gather_pull|pull_rows" | head -4
  done
done
