python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -m gpu 2>&1 | tail -2
echo "== min blocks 2"; timeout 600 python tools/apsp_probe.py --k 512 --single 4 2>&1 | grep -v "^ *[0-9]"
echo "== min blocks 3"; DAWN_LIB=paper_2306_07872_b200/libdawn_b3.so timeout 600 python tools/apsp_probe.py --k 512 --single 4 2>&1 | grep -v "^ *[0-9]"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dawn_batch_persistent -s 3 -c 1 -o gpurun_out/prof_batch3 -f python tools/apsp_probe.py --k 128 --single 2 > gpurun_out/ncu_batch.log 2>&1; echo "ncu rc=$?"
