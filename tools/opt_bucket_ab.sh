python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
[ -n "${SKIPTEST:-}" ] || timeout 900 python -m pytest tests/test_gpu_ep.py tests/test_gpu_optim.py -q -k "sharded_optimizer or optim" 2>&1 | tail -2
for b in 1 8 4; do
  echo "== B2_OPT_BUCKETS=$b"
  B2_OPT_BUCKETS=$b timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955$b bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu --zipf 0 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); a=d['adamw']; b=d['adamw_dp_axis']
        print('ep axis', a['parallelism'], round(a['ms'],2), 'ms  roof/meas', round(a['roofline_over_measured'],3), '| dp axis', b['parallelism'], round(b['ms'],2), 'ms roof/meas', round(b['roofline_over_measured'],3))
"
done
