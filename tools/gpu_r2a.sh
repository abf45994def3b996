#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep_dist.py -x -q -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "exit $?" >> gpurun_out/pytest_dist.log
timeout 900 python bench.py --no-layer-step > gpurun_out/bench1.log 2>&1; echo "exit $?" >> gpurun_out/bench1.log
timeout 900 python bench.py --gpus 2 --no-layer-step --no-e2e > gpurun_out/bench2.log 2>&1; echo "exit $?" >> gpurun_out/bench2.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
