python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "small-cta or golden_cases" 2>&1 | tail -1
for lib in default base default base; do if [ $lib = default ]; then unset DAWN_LIB; else export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_$lib.so; fi; echo "== $lib"; python tools/small_probe.py 2>&1 | grep cluster; done
