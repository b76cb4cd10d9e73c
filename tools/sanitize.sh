#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (the B200 analogue of the reference's collective
# deadlock / mismatch checks, comm.cpp:139-176, 240-250): memcheck, racecheck (shared memory),
# synccheck (barriers) and initcheck on one GPU; memcheck on the EP = 2 peer-memory path.
# Usage on the GPU box: bash tools/sanitize.sh OUTDIR [ep2]
OUT=${1:-gpurun_out/sanitize}; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case ok' $OUT/$tool.log | tr '\n' ' ')"
done
if [ "${2:-}" = "ep2" ]; then
  timeout 1200 $CS --tool memcheck --print-limit 50 --error-exitcode 9 --target-processes all \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    tools/sanitize_case.py > $OUT/memcheck_ep2.log 2>&1
  echo "memcheck ep2 rc=$? $(grep -E 'ERROR SUMMARY|layer ok' $OUT/memcheck_ep2.log | tr '\n' ' ')"
fi
