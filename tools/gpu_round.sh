#!/bin/bash
# One GPU session: gpu tests, smoke, bench line, launch list, ncu --set full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_replay.py 48 > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 2 -c 1 -o gpurun_out/replay_full -f python tools/ncu_replay.py 48 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_persistent -s 32 -c 1 -o gpurun_out/router_full -f python tools/ncu_replay.py 8 > gpurun_out/ncu_router.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_decode_kernel -s 5 -c 1 -o gpurun_out/ffn_decode_full -f python tools/bench_ffn.py > gpurun_out/ncu_ffn1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_fused -s 5 -c 1 -o gpurun_out/ffn_prefill_full -f python tools/bench_ffn.py > gpurun_out/ncu_ffn2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_decode_q -s 9 -c 1 -o gpurun_out/ffn_decode_q_full -f python tools/bench_ffn.py > gpurun_out/ncu_ffn3.log 2>&1
timeout 300 python tools/bench_ffn.py > gpurun_out/bench_ffn.log 2>&1
echo done
