python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_async.py -x -q -m gpu > gpurun_out/pytest_async.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/pytest_async.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/pytest_gpu.log
