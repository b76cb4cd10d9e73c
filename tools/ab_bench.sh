#!/bin/bash
# Same-box A/B of the 1-GPU layer step: alternates the in-tree build and build/ab/<name>.so
# (tools/ab_build.sh) ROUNDS times and prints each run's ms_per_step and per-stage times.
#   bash tools/ab_bench.sh base [ROUNDS]
NAME=$1; ROUNDS=${2:-2}
for i in $(seq $ROUNDS); do
  for lib in "" "build/ab/$NAME.so"; do
    B2_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-adamw --no-cpu --no-parity --zipf 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${lib:-tree}'.ljust(22), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stage_ms'].items()})"
  done
done
