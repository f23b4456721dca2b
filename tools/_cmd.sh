#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for t in 0 131072 1048576; do
  echo "== worklist_edges=$t"
  timeout 300 python tools/round_profile.py --solves 7 --tune worklist_edges=$t > gpurun_out/wl_$t.txt 2>&1; head -1 gpurun_out/wl_$t.txt; grep "worklist:\|after the last" gpurun_out/wl_$t.txt
done
