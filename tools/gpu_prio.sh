# Priority-window A/B on one box: C2 rounds under several solver tunings (TUNES: space-separated
# "key=value,key=value" sets; "-" = defaults), the HEAD-before library (DAWN_LIB=base, if present),
# and the async / parity / scale GPU tests (TESTS=0 skips them).
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  if [ -f paper_2306_07872_b200/libdawn_base.so ]; then
    echo "== base"; DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_base.so timeout 300 python tools/round_profile.py --solves 7 2>&1 | grep "solve ms\|sum S"
  fi
  for t in ${TUNES:--}; do
    args=""; [ "$t" != "-" ] && for kv in ${t//,/ }; do args="$args --tune $kv"; done
    echo "== $t"; timeout 300 python tools/round_profile.py --solves 7 $args 2>&1 | grep "solve ms\|sum S"
  done
done
timeout 300 python tools/round_profile.py --solves 3 2>&1 | head -20
[ "${TESTS:-1}" = 1 ] && timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_parity.py tests/test_gpu_worklist.py tests/test_gpu_scale.py -x -q 2>&1 | tail -3
