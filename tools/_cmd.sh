#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python tools/e2e_probe.py
bash tools/gpu_check.sh tests
