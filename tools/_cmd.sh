#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in new old; do
  if [ $v = old ]; then export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_old.so; else unset DAWN_LIB; fi
  timeout 900 python tools/bench_configs.py --only c4 --solves 3 > gpurun_out/c4_$v.txt 2>&1; echo "== $v"; python -c "
import json,sys
for l in open('gpurun_out/c4_$v.txt'):
    if l.startswith('{'):
        r=json.loads(l); print(r['config'], r['ms_median'], r['async_ms_median'], r['parity'])"
done
