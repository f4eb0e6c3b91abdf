# Cost of the fused step's scatter parts (experiment builds, wrong results by construction):
# x5 = no packed x-halo writes, x6 = no y/z face writes, x7 = no y face rows, x8 = no z face planes.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e10_base.json 2>/dev/null
for v in ${VARIANTS:-5 6 7 8}; do TILEMESH_LIB=$PWD/build/var/lib_x$v.so $B > gpurun_out/e10_x$v.json 2>/dev/null; done
