set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_mu.py -x -q > gpurun_out/batch_tests.log 2>&1; echo "batch tests rc=$?"; tail -3 gpurun_out/batch_tests.log
for u in 4; do echo "== util $u"; timeout 300 python tools/apsp_probe.py --k 512 --single 4 --util $u 2>&1 | head -1; done
timeout 300 python tools/apsp_probe.py --k 512 --single 4 2>&1 | tail -30
