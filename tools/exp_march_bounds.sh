# Timing experiments on the fused C2 step: data-movement-only (x1), no-store (x2)
# and no-x-halo-copy (x3) builds of the march kernel (wrong results by
# construction) against the real one.
B="python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-pipeline"
$B > gpurun_out/e2_base.json 2>gpurun_out/e2_base.err
for v in ${VARIANTS:-1 2 3}; do TILEMESH_LIB=$PWD/build/var/lib_x$v.so $B > gpurun_out/e2_x$v.json 2>gpurun_out/e2_x$v.err; done
