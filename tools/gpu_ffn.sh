#!/bin/bash
# Decode FFN session: FFN + layer-step GPU tests, the FFN microbenchmark.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_layer_step.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_ffn.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ffn.log
timeout 600 python tools/bench_ffn.py > gpurun_out/bench_ffn.log 2>&1; echo "bench_ffn exit $?" >> gpurun_out/bench_ffn.log
echo done
