# A/B on one box: the working tree's libdawn.so vs a variant (DAWN_LIB) on C2 rounds and C3
set -u
v=${1:-base}; w=${2:-}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  for lib in default $v $w; do
    if [ $lib = default ]; then unset DAWN_LIB; else export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_$lib.so; fi
    echo "== $lib"
    [ "${SKIP_C2:-0}" = 1 ] || timeout 300 python tools/round_profile.py --solves 7 2>&1 | grep "solve ms\|sum S"
    [ "${SKIP_C3:-0}" = 1 ] || timeout 300 python tools/apsp_probe.py --k 512 --single 2 2>&1 | grep "batched\|sum B"
  done
done
