#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python tools/round_profile.py --solves 9 > gpurun_out/rp_$i.txt 2>&1; head -1 gpurun_out/rp_$i.txt; grep "sum S" gpurun_out/rp_$i.txt; sed -n 3,4p gpurun_out/rp_$i.txt; done
timeout 300 python tools/apsp_probe.py --k 1024 --single 2 2>&1 | head -1
