#!/bin/bash
# One gpurun round: GPU tests, smoke, 1-GPU bench, ncu launch list, ncu --set full of the GEMMs.
# Usage (from this container): gpurun --timeout 1800 -- 'bash tools/gpu_check.sh TAG [what...]'
# what ∈ {tests, smoke, bench, launches, full, ep2}; default: all but ep2.
set -u
TAG=${1:-run}; shift || true
WHAT=${*:-tests smoke bench launches full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
for w in $WHAT; do case $w in
 tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log ;;
 smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log ;;
 bench) timeout 600 python bench.py --steps 20 --warmup 5 --profile > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -20 $OUT/bench.err ;;
 benchq) timeout 300 python bench.py --steps 20 --warmup 5 --profile --no-adamw --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -20 $OUT/bench.err ;;
 launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-adamw --no-cpu > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?" ;;
 full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel --launch-skip 16 -c 8 \
      -o $OUT/gemm_full python bench.py --steps 1 --warmup 3 --no-adamw --no-cpu > $OUT/ncu_full.log 2>&1; echo "full rc=$?"; tail -3 $OUT/ncu_full.log ;;
 fullk) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" --launch-skip ${KSKIP:-4} -c ${KCOUNT:-1} \
      -o $OUT/k_full python bench.py --steps 1 --warmup 3 --no-adamw --no-cpu > $OUT/ncu_fullk.log 2>&1; echo "fullk rc=$?"; tail -3 $OUT/ncu_fullk.log ;;
 ep2) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/ep2.json 2> $OUT/ep2.err; echo "ep2 rc=$?"; cat $OUT/ep2.json; tail -5 $OUT/ep2.err ;;
 timeline) timeout 300 python tools/timeline.py > $OUT/timeline_eager.txt 2>&1; echo "timeline rc=$?"; head -30 $OUT/timeline_eager.txt
      timeout 300 python tools/timeline.py --graph > $OUT/timeline_graph.txt 2>&1; head -30 $OUT/timeline_graph.txt ;;
 tl2) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/timeline.py --graph 2>&1 | grep -v "Warn\|warn\|\*\*\*\|OMP" | head -45 ;;
 tl4) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/timeline.py --graph 2>&1 | grep -v "Warn\|warn\|\*\*\*\|OMP" | head -45 ;;
 ckpt) timeout 600 python -m pytest tests/test_gpu_ckpt.py tests/test_records.py -x -q > $OUT/ckpt_tests.log 2>&1; echo "ckpt tests rc=$?"; tail -15 $OUT/ckpt_tests.log
      timeout 300 python tools/ckpt_probe.py --dir /tmp > $OUT/ckpt_probe.json 2> $OUT/ckpt_probe.err; echo "probe rc=$?"; cat $OUT/ckpt_probe.json; tail -3 $OUT/ckpt_probe.err ;;
 adamw) timeout 300 python tools/adamw_probe.py --gelems 2 > $OUT/adamw.txt 2>&1; cat $OUT/adamw.txt
      timeout 600 ncu --set full --clock-control none -k regex:"adamw_chunks|sumsq_chunks" --launch-skip 2 -c 2 -o $OUT/adamw_full python tools/adamw_probe.py --gelems 0.5 --steps 1 > $OUT/ncu_adamw.log 2>&1; echo "adamw ncu rc=$?" ;;
 gtest) timeout 600 python -m pytest tests -m gpu -x -q -k "${GTEST_K}" > $OUT/gtest.log 2>&1; echo "gtest rc=$?"; tail -15 $OUT/gtest.log ;;
 ep4) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus 4 --steps 10 --warmup 3 > $OUT/ep4.json 2> $OUT/ep4.err; echo "ep4 rc=$?"; cat $OUT/ep4.json; tail -5 $OUT/ep4.err ;;
 ref) timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"; cat $OUT/ref.json ;;
esac; done
