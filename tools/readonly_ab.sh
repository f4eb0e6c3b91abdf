for S in 4 8 12; do
  sed -i "s/constexpr int kStages = [0-9]*;/constexpr int kStages = $S;/" paper_1604_03570_b200/csrc/tm_march.cu
  sed -i "s/^STAGES = [0-9]*/STAGES = $S/" paper_1604_03570_b200/march.py
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -DTM_MARCH_COPY_EXPERIMENT -DTM_EXP_NOSTORE -o build/lib_ro_$S.so paper_1604_03570_b200/csrc/*.cu 2>/dev/null
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -DTM_MARCH_COPY_EXPERIMENT -o build/lib_cp_$S.so paper_1604_03570_b200/csrc/*.cu 2>/dev/null
  echo "=== stages $S read-only"; TILEMESH_LIB=$PWD/build/lib_ro_$S.so timeout -s KILL 600 python tools/march_perf.py --noscatter 2>&1 | grep noscatter
  echo "=== stages $S copy"; TILEMESH_LIB=$PWD/build/lib_cp_$S.so timeout -s KILL 600 python tools/march_perf.py --noscatter 2>&1 | grep noscatter
done
