cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/probe_points.py 48 > gpurun_out/points.json 2> gpurun_out/points.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 3 -c 3 -o gpurun_out/replay_src -f python tools/ncu_replay.py 48 > gpurun_out/ncu_src.log 2>&1
echo done
