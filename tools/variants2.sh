#!/bin/bash
# build replay variants from -D flag sets ($VARIANTS, ';'-separated) and time the C5 x 48 replay
set -e
cd $GRAFT_REPO_ROOT
IFS=';' read -ra VS <<< "${VARIANTS}"
i=0
for V in "${VS[@]}"; do
  D=/tmp/var$i; mkdir -p $D; i=$((i+1))
  for f in capi router replay ffn_gemm layer_step policy report; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $V -c paper_2602_03921_b200/csrc/$f.cu -o $D/$f.o 2>&1 | grep -E "error" || true
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/lib.so $D/*.o -lcudart
  echo "variant [$V]"
  ESIM_LIB=$D/lib.so python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from bench import make_traces
from paper_2602_03921_b200.sweep import DeviceSweep, c5_points
cfgs, trs = c5_points(make_traces(list(range(1, 49))))
ds = DeviceSweep(cfgs, trs)
ds.step(); torch.cuda.synchronize()
ds.tune_order(); ds.step(); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ds.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
res = ds.results()
acc = sum(r.counters.totals[0] for r in res)
print(f"   replay_ms={min(ts):.1f} acc/s={acc/(min(ts)/1e3)/1e6:.1f}M  digest0={res[0].counters.digest:#x}", flush=True)
PY
done
