#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/round_profile.py --solves 7 > gpurun_out/rounds_c2.txt 2>&1; head -1 gpurun_out/rounds_c2.txt; grep "sum S" gpurun_out/rounds_c2.txt
grep -A 11 "S min" gpurun_out/rounds_c2.txt
