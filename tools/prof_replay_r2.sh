#!/bin/bash
# replay kernel: per-point times + one ncu --set full capture of each policy launch (source-level)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_points.py 48 > gpurun_out/points.json 2> gpurun_out/points.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 3 -c 3 -o gpurun_out/replay_src -f python tools/ncu_replay.py 16 > gpurun_out/ncu_src.log 2>&1
python tools/ncu_src_hot.py gpurun_out/replay_src.ncu-rep 60 > gpurun_out/replay_hot.txt 2>&1
python tools/ncu_summary.py gpurun_out/replay_src.ncu-rep gpurun_out/replay_summary.json > /dev/null 2>&1
echo done
