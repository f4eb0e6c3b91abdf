# C4 GSRB colour-split pass timing + parity tests
timeout 300 python tools/gsrb_perf.py > gpurun_out/e4_gsrb_perf.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_march.py -x -q -k "gsrb or c4" > gpurun_out/e4_pytest.log 2>&1
timeout 600 python tools/run_configs.py C4 --oracle > gpurun_out/e4_c4.jsonl 2>&1
