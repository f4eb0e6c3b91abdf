# Fused C2 step with the x-halo scatter as one predicated 16-B store per lane (product build)
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e11_a.json 2>/dev/null
$B > gpurun_out/e11_b.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q > gpurun_out/e11_pytest.log 2>&1
