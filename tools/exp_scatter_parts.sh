# Cost of the fused step's scatter parts: x5 = no packed x-halo writes, x6 = no y/z face
# writes (experiment builds, wrong results by construction), fused C2 step.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e10_base.json 2>/dev/null
for v in 5 6; do TILEMESH_LIB=$PWD/build/var/lib_x$v.so $B > gpurun_out/e10_x$v.json 2>/dev/null; done
