for S in 4 6 8; do
  sed -i "s/constexpr int kStages = [0-9]*;/constexpr int kStages = $S;/" paper_1604_03570_b200/csrc/tm_march.cu
  sed -i "s/^STAGES = [0-9]*/STAGES = $S/" paper_1604_03570_b200/march.py
  python -c "from paper_1604_03570_b200._build import build_library; build_library(force=True)"
  echo "=== stages $S"; timeout -s KILL 600 python tools/march_perf.py 2>&1 | grep fused | grep -E "rows=(16|8)"
done
