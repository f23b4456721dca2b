#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_worklist.py tests/test_gpu_async.py tests/test_oracles_device.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for wl in 0 131072 524288 1048576 4194304; do
  timeout 300 python tools/round_profile.py --solves 9 --tune worklist_edges=$wl > gpurun_out/wl_$wl.txt 2>&1; echo "== wl=$wl"; head -1 gpurun_out/wl_$wl.txt; grep "worklist:" gpurun_out/wl_$wl.txt
done
