#!/bin/bash
# replay kernel: one ncu --set full capture of the three policy launches (C5 x 16), reduced to code regions
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 3 -c 3 -o gpurun_out/replay_c5 -f python tools/ncu_replay.py 16 > gpurun_out/ncu_c5.log 2>&1
python tools/region_profile.py gpurun_out/replay_c5.ncu-rep > gpurun_out/replay_regions_c5.txt 2>&1
ncu -i gpurun_out/replay_c5.ncu-rep --page details --csv > gpurun_out/replay_c5_details.csv 2>&1
rm -f gpurun_out/replay_c5.ncu-rep
