#!/bin/bash
# quantised decode FFN A/B: production build vs diagnostic builds (lib/variants/libq_<name>.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2602_03921_b200/lib/libspecmd_b200.so /tmp/base.so
for v in base "$@"; do
  if [ "$v" = base ]; then cp /tmp/base.so paper_2602_03921_b200/lib/libspecmd_b200.so;
  else cp paper_2602_03921_b200/lib/variants/libq_$v.so paper_2602_03921_b200/lib/libspecmd_b200.so; fi
  echo "== $v" >> gpurun_out/ffnq_var.log
  timeout 300 python tools/bench_ffn.py 2>&1 | grep -E "^decode" | cut -c1-60 >> gpurun_out/ffnq_var.log
done
