for h in 0 1 2 3; do echo "TMA_HINT=$h"; TM_TMA_HINT=$h timeout -s KILL 300 python tools/sweep_shapes.py 2>&1 | sed -n 2,3p; done
python tools/c2_steps.py 4 > gpurun_out/plain.log 2>&1 && TM_TMA_HINT=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:"heat_vec" -c 1 python tools/c2_steps.py 4 2>&1 | grep -E "dram__|lts__|duration"
