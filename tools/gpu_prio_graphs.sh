# Priority window on / off on other RMAT shapes (C2's neighbours): async solve times and relaxations.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spec in "--scale 22 --ef 16 --weights int --precision auto" "--scale 20 --ef 16" "--scale 22 --ef 8" "--scale 23 --ef 16" "--scale 21 --ef 32"; do
  for t in "" "--tune priority_frac=0"; do
    echo "== $spec $t"; timeout 300 python tools/round_profile.py $spec --solves 5 $t 2>&1 | grep "solve ms"
  done
done
