# C4 GSRB colour-split pass timing: column heights x CTAs per SM (profiles/gsrb_split_shapes_r01.txt)
for r in 16 32; do for n in 148 296; do echo "rows=$r nctas=$n: $(timeout 300 python tools/gsrb_perf.py --rows $r --nctas $n 2>&1 | tail -1)"; done; done > gpurun_out/e5_gsrb.txt
timeout 600 python -m pytest tests/test_gpu_march.py -x -q -k "split" > gpurun_out/e5_pytest.log 2>&1
