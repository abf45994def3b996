cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ESIM_PROFILE_HOST=1 timeout 300 python tools/probe_e2e.py > gpurun_out/probe_e2e.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_kernels.csv python tools/ncu_replay.py 48 > gpurun_out/step_ncu.log 2>&1
echo ok
