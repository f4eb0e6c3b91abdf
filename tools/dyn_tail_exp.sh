# The dynamic-tail experiment (profiles/r02/dynamic_tail_prefetch_experiment.diff applied): parity under a pool, then C2 step times per pool size / chunk.
set -x
TM_MARCH_POOL=10 TM_MARCH_CHUNK=4 python -m pytest tests/test_gpu_march.py -m gpu -x -q -k "fused_runner or std_matches" 2>&1 | tail -3
TM_MARCH_POOL=5 TM_MARCH_CHUNK=2 python -m pytest tests/test_gpu_production.py -m gpu -x -q -k "c2 or C2" 2>&1 | tail -3
for rep in 1 2; do
python tools/march_exp.py --reps 200 | tail -1
for pc in 3:2 5:2 5:3 5:4 8:2 8:4 10:4 10:8 15:4; do
  P=${pc%%:*}; C=${pc##*:}
  echo "pool $P chunk $C"; TM_MARCH_POOL=$P TM_MARCH_CHUNK=$C python tools/march_exp.py --reps 200 | tail -1
done
done
