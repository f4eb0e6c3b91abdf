set -x
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
for pdl in 0 1; do TM_PDL=$pdl $B > gpurun_out/e1_s4_pdl$pdl.json 2>gpurun_out/e1_s4_pdl$pdl.err; done
for pdl in 0 1; do TM_PDL=$pdl TM_HEAT_STAGES=8 TILEMESH_LIB=$PWD/build/var/lib_s8.so $B > gpurun_out/e1_s8_pdl$pdl.json 2>gpurun_out/e1_s8_pdl$pdl.err; done
TM_PDL=1 timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_parity.py -x -q > gpurun_out/e1_pytest.log 2>&1
tail -2 gpurun_out/e1_pytest.log
