python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 2400 python tools/bench_configs.py --out gpurun_out/configs.json 2>&1 | tail -12
