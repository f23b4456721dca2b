set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_batch.py tests/test_gpu_worklist.py -x -q 2>&1 | tail -2
timeout 300 python tools/round_profile.py --solves 5 2>&1 | head -17
timeout 300 python tools/apsp_probe.py --k 512 --single 4 2>&1 | grep "batched\|sum B"
