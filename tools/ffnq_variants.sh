#!/bin/bash
# quantised decode FFN: GPU tests (FFN + layer step) and the microbenchmark
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_layer_step.py -q -p no:cacheprovider -x > gpurun_out/pytest_ffn.log 2>&1
timeout 300 python tools/bench_ffn.py > gpurun_out/bench_ffn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_decode_q -s 66 -c 1 -o gpurun_out/ffn_q4 -f python tools/bench_ffn.py > gpurun_out/ncu_q4.log 2>&1
python tools/ncu_summary.py gpurun_out/ffn_q4.ncu-rep gpurun_out/ffn_q4_summary.json > /dev/null 2>&1
