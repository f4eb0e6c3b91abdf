for c in 1 2 4 8; do echo "CLUSTER=$c"; TM_CLUSTER=$c timeout -s KILL 300 python tools/sweep_shapes.py 2>&1 | sed -n 2,4p; done
python tools/c2_steps.py 4 > gpurun_out/plain.log 2>&1 && TM_CLUSTER=8 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:"heat_vec" -c 2 python tools/c2_steps.py 4 2>&1 | grep -E "dram__|lts__|duration"
