# Fused C2 step: y/z halos read from the neighbour boxes (NBRH, default) vs scattered into
# the ghosts of unew (TM_NBRH=0); then the GPU parity suites with NBRH on.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e12_nbrh.json 2>gpurun_out/e12_nbrh.err
TM_NBRH=0 $B > gpurun_out/e12_scatter.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_regional.py -x -q > gpurun_out/e12_pytest.log 2>&1
timeout 300 python tools/run_configs.py C3 C5 > gpurun_out/e12_configs.jsonl 2>&1
