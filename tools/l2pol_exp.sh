#!/bin/bash
# C2 fused step under the L2 eviction-policy switches of the march (TM_L2POL bits: 1 = plane
# loads evict_first, 2 = cell stores with a policy, 4 = that policy is evict_first, else evict_last)
for pol in 0 1 2 3 6 7 0; do
  echo "TM_L2POL=$pol"
  TM_L2POL=$pol python tools/march_exp.py --config C2 --reps 200 2>&1 | tail -2
done
for cfg in C3 C5; do for pol in 0 3; do echo "$cfg TM_L2POL=$pol"; TM_L2POL=$pol python tools/march_exp.py --config $cfg --reps 10 2>&1 | tail -1; done; done
