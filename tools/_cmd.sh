python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_mu.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for u in 0 2 4 6 10 33; do echo "== util $u"; timeout 600 python tools/apsp_probe.py --k 512 --single 2 --util $u 2>&1 | grep -E "^batched|sum B"; done
