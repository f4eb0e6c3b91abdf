# Ring depth 4 vs 8 for the product kernel and the x1 (data movement only) / x2 (no stores)
# experiment builds (wrong results by construction), fused C2 step.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e6_s4.json 2>/dev/null
TM_HEAT_STAGES=8 TILEMESH_LIB=$PWD/build/var/lib_s8.so $B > gpurun_out/e6_s8.json 2>/dev/null
for v in 1 2; do
  TILEMESH_LIB=$PWD/build/var/lib_x$v.so $B > gpurun_out/e6_x${v}_s4.json 2>/dev/null
  TM_HEAT_STAGES=8 TILEMESH_LIB=$PWD/build/var/lib_x${v}_s8.so $B > gpurun_out/e6_x${v}_s8.json 2>/dev/null
done
