#!/bin/bash
# A/B of the in-tree library against libb2moe_alt.so (tools/build_alt.sh) on one box, alternating.
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_moe.py tests/test_gpu_golden.py -q -x 2>&1 | tail -1
for i in 1 2; do for L in alt default; do
  if [ $L = alt ]; then export B2_LIB=paper_2604_00785_b200/libb2moe_alt.so; else unset B2_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-adamw --no-cpu --zipf 0 --profile 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); st=d['stage_ms']; print('$L', round(d['ms_per_step'],3), ' '.join(f'{k[:10]}={v:.3f}' for k,v in st.items()))"
done; done
