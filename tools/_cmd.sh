#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in base exp base exp; do
  if [ $v = exp ]; then export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_exp.so; else unset DAWN_LIB; fi
  timeout 300 python tools/round_profile.py --solves 5 > gpurun_out/ns_$v.txt 2>&1; echo "== $v"; sed -n 3,6p gpurun_out/ns_$v.txt
done
