#!/bin/bash
# One GPU session: gpu tests, smoke, bench line, launch list, ncu --set full captures of the hot kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
# launch list of the bench's own command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-layer-step > gpurun_out/b_ncu.log 2>&1
# per-step traffic + instruction totals of the replay launches (C5 x 48)
timeout 900 ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:replay_kernel --clock-control none --csv --log-file gpurun_out/replay_traffic.csv python tools/ncu_replay.py 48 > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 3 -c 3 -o gpurun_out/replay_full -f python tools/ncu_replay.py 16 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/replay_full.ncu-rep gpurun_out/replay_full_summary.json > /dev/null 2>&1
python tools/region_profile.py gpurun_out/replay_full.ncu-rep > gpurun_out/replay_regions.txt 2>&1
rm -f gpurun_out/replay_full.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_decode_kernel -s 5 -c 1 -o gpurun_out/ffn_decode_full -f python tools/bench_ffn.py > gpurun_out/ncu_ffn1.log 2>&1
python tools/ncu_summary.py gpurun_out/ffn_decode_full.ncu-rep gpurun_out/ffn_decode_summary.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_fused -s 5 -c 1 -o gpurun_out/ffn_prefill_full -f python tools/bench_ffn.py > gpurun_out/ncu_ffn2.log 2>&1
python tools/ncu_summary.py gpurun_out/ffn_prefill_full.ncu-rep gpurun_out/ffn_prefill_summary.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_persistent -s 32 -c 1 -o gpurun_out/router_full -f python tools/ncu_replay.py 8 > gpurun_out/ncu_router.log 2>&1
python tools/ncu_summary.py gpurun_out/router_full.ncu-rep gpurun_out/router_summary.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_gemv --launch-skip 92 --launch-count 1 -o gpurun_out/ffn_gemv_full -f python tools/probe_gemv_variants.py paper_2602_03921_b200/lib/libspecmd_b200.so > gpurun_out/ncu_gemv.log 2>&1
python tools/ncu_summary.py gpurun_out/ffn_gemv_full.ncu-rep gpurun_out/ffn_gemv_summary.json > /dev/null 2>&1
timeout 300 python tools/bench_ffn.py > gpurun_out/bench_ffn.log 2>&1
timeout 300 python tools/probe_gemv_variants.py paper_2602_03921_b200/lib/libspecmd_b200.so > gpurun_out/pgv.log 2>&1
rm -f gpurun_out/*.ncu-rep
echo done
