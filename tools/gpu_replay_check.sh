#!/bin/bash
# replay kernel change: parity tests (goldens, fuzz, host semantics, sharded), then the headline bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_acceptance.py tests/test_host_semantics.py tests/test_gpu_sweep_dist.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/pytest_replay.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_replay.log
timeout 900 python bench.py --no-layer-step > gpurun_out/bench_replay.log 2>&1
