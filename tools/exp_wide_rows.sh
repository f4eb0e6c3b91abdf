# PACKED plane rows staged 16 doubles wider on each side (whole 768-B pitch rows, 1.5x the
# bytes) vs exact 512-B rows, product and no-store builds, fused C2 step.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e8_base.json 2>/dev/null
TILEMESH_LIB=$PWD/build/var/lib_w16.so $B > gpurun_out/e8_w16.json 2>/dev/null
TILEMESH_LIB=$PWD/build/var/lib_x2.so $B > gpurun_out/e8_x2.json 2>/dev/null
TILEMESH_LIB=$PWD/build/var/lib_x2_w16.so $B > gpurun_out/e8_x2_w16.json 2>/dev/null
TILEMESH_LIB=$PWD/build/var/lib_w16.so timeout 600 python -m pytest tests/test_gpu_march.py -x -q > gpurun_out/e8_pytest.log 2>&1
