#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${MODELS:-mixtral olmoe}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 3 -c 3 -o gpurun_out/replay_$m -f python tools/ncu_replay_model.py $m 16 > gpurun_out/ncu_$m.log 2>&1
  python tools/region_profile.py gpurun_out/replay_$m.ncu-rep > gpurun_out/replay_regions_$m.txt 2>&1
  python tools/ncu_summary.py gpurun_out/replay_$m.ncu-rep gpurun_out/replay_summary_$m.json > /dev/null 2>&1
  rm -f gpurun_out/replay_$m.ncu-rep
done
