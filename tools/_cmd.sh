#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in 0 1 2 3 5 99; do
  timeout 300 python tools/round_profile.py --solves 7 --tune l2_gather_rounds=$c > gpurun_out/cg_$c.txt 2>&1; echo "== cg=$c"; head -1 gpurun_out/cg_$c.txt; sed -n 3,10p gpurun_out/cg_$c.txt
done
