# C4 GSRB colour-split pass timing: column heights, warps x rows, CTAs per SM
for r in 16 32; do for n in 148 296; do echo "rows=$r nctas=$n: $(timeout 300 python tools/gsrb_perf.py --rows $r --nctas $n 2>&1 | tail -1)"; done; done > gpurun_out/e5_gsrb.txt
for n in 148 296; do echo "rows=32 rpw4 nctas=$n: $(TM_SPLIT_RPW4=1 timeout 300 python tools/gsrb_perf.py --rows 32 --nctas $n 2>&1 | tail -1)"; done >> gpurun_out/e5_gsrb.txt
TM_SPLIT_RPW4=1 timeout 600 python -m pytest tests/test_gpu_march.py -x -q -k "split" > gpurun_out/e5_pytest.log 2>&1
