#!/bin/bash
# build replay variants with different register caps and time the C5 x 48 replay
set -e
cd $GRAFT_REPO_ROOT
for MINB in ${MINBS:-1 2 3}; do
  D=/tmp/v$MINB; mkdir -p $D
  for f in capi router replay ffn_gemm layer_step policy; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DESIM_SIMPLE_MINB=$MINB -c paper_2602_03921_b200/csrc/$f.cu -o $D/$f.o 2>&1 | grep -E "error" || true
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/lib.so $D/*.o -lcudart
  cuobjdump -res-usage $D/lib.so 2>/dev/null | grep -A1 "replay_kernelILi5ELi0" | grep -oE "REG:[0-9]+|STACK:[0-9]+|LOCAL:[0-9]+" | tr '\n' ' '
  echo " minb=$MINB"
  ESIM_LIB=$D/lib.so python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
for wpc in (0, 3):
    ds.batch.launch(warps_per_cta=wpc); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.batch.launch(warps_per_cta=wpc); e1.record(); torch.cuda.synchronize()
    res = ds.results()
    acc = sum(r.counters.totals[0] for r in res)
    print(f"   wpc={wpc} replay_ms={e0.elapsed_time(e1):.1f} acc/s={acc/(e0.elapsed_time(e1)/1e3)/1e6:.1f}M", flush=True)
PY
done
