#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in base xi12 base xi12; do
  if [ $v = xi12 ]; then export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_xi12.so; else unset DAWN_LIB; fi
  timeout 300 python tools/round_profile.py --solves 9 > gpurun_out/x_$v.txt 2>&1; echo "== $v"; head -1 gpurun_out/x_$v.txt; grep "sum S" gpurun_out/x_$v.txt
done
