set -u
OUT=gpurun_out/${TAG:-s18}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
[ -n "${SKIPTEST:-}" ] || timeout 600 python -m pytest tests/test_gpu_ep.py -x -q -k "ep_matches" > $OUT/eptests.log 2>&1; echo "ep tests rc=$?"; tail -5 $OUT/eptests.log
for fp in 0 1 0 1; do
  echo "== B2_EP_FUSED_PULL=$fp"
  B2_EP_FUSED_PULL=$fp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$fp tools/timeline.py --graph 2>&1 | grep -E "event-timed|grouped_gemm|gather_pull|out_reduction|tile_" | head -8
done
