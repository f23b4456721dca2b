#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_oracles_device.py -x -q > gpurun_out/pytest_or.log 2>&1; echo "oracles rc=$?"; tail -15 gpurun_out/pytest_or.log
timeout 600 python tools/fw_probe.py 2>&1 | tail -4
