#!/bin/bash
# A/B of replay-kernel build variants (lib/variants/lib_<name>.so) on the headline bench (device leg)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2602_03921_b200/lib/libspecmd_b200.so /tmp/base.so
for v in base "$@"; do
  if [ "$v" = base ]; then cp /tmp/base.so paper_2602_03921_b200/lib/libspecmd_b200.so;
  else cp paper_2602_03921_b200/lib/variants/lib_$v.so paper_2602_03921_b200/lib/libspecmd_b200.so; fi
  echo "== $v" >> gpurun_out/replay_var.log
  timeout 600 python bench.py --no-layer-step --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']/1e6,1), 'M acc/s', d['kernel_ms'], 'tuned', round(d['value_tuned_order']['value']/1e6,1), d['parity'])
" >> gpurun_out/replay_var.log
done
