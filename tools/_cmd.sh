#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_distributed.py tests/test_gpu_mu.py -x -q > gpurun_out/pytest_b.log 2>&1; echo "batch rc=$?"; tail -3 gpurun_out/pytest_b.log
for sch in jacobi async; do
  timeout 300 python tools/apsp_probe.py --k 2048 --single 4 --schedule $sch > gpurun_out/apsp_$sch.txt 2>&1; echo "== $sch"; head -8 gpurun_out/apsp_$sch.txt
done
