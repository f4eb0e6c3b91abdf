# MultiFab rows aligned to 64 B (TM_ROW_ALIGN=8: pitch 80, first valid column 8) vs 128 B
# (pitch 96, column 16), fused C2 step, with the GPU parity suites under the 64-B layout.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
TILEMESH_LIB=$PWD/build/var/lib_x2.so $B > gpurun_out/e9_x2_a16.json 2>/dev/null
$B > gpurun_out/e9_a16.json 2>/dev/null
TM_ROW_ALIGN=8 TILEMESH_LIB=$PWD/build/var/lib_a8.so $B > gpurun_out/e9_a8.json 2>/dev/null
TM_ROW_ALIGN=8 TILEMESH_LIB=$PWD/build/var/lib_x2_a8.so $B > gpurun_out/e9_x2_a8.json 2>/dev/null
TM_ROW_ALIGN=8 TILEMESH_LIB=$PWD/build/var/lib_a8.so timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_parity.py -x -q > gpurun_out/e9_pytest.log 2>&1
