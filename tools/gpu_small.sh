set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_worklist.py tests/test_gpu_nearfar.py tests/test_gpu_cabi.py -x -q 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --only c1 --solves 9 > gpurun_out/configs.txt 2>&1
python -c "
import json
for l in open('gpurun_out/configs.txt'):
    if l.startswith('{'):
        r=json.loads(l); print(r['config'], 'jacobi', r['ms_all'], 'async', round(r['async_ms_median'],4), r['parity'])"
tail -3 gpurun_out/configs.txt
