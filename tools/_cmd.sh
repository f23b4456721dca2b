#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_worklist.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for fb in 0 1; do for wl in 131072 0; do
  timeout 300 python tools/round_profile.py --solves 7 --tune bitmap_frontier=$fb --tune worklist_edges=$wl > gpurun_out/fb${fb}_wl$wl.txt 2>&1; echo "== C2 fb=$fb wl=$wl"; head -1 gpurun_out/fb${fb}_wl$wl.txt; grep "sum S\|worklist:" gpurun_out/fb${fb}_wl$wl.txt
done; done
for wl in 0 131072 1048576 1e12; do
  timeout 300 python tools/round_profile.py --solves 3 --grid 2048 --tune worklist_edges=$wl > gpurun_out/grid_wl$wl.txt 2>&1; echo "== grid2048 fb=auto wl=$wl"; head -1 gpurun_out/grid_wl$wl.txt; grep "worklist:" gpurun_out/grid_wl$wl.txt
done
