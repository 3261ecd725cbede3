# Resident-kernel phase stamps of the four C2 orders after a 512 MiB L2 flush (as bench.py)
O=gpurun_out/${1:-stamps}
mkdir -p $O
for o in random few_unique nearly reversed; do
  echo "== $o"
  SR_TIMING=1 timeout 120 python tools/profile_one.py --order $o --warmup 3 --flush > $O/x.log 2>&1
  grep -E "route step|phases|C splitters|C.route|C.tree|C.end|D.end|E.end|E items|last sort" $O/x.log | tail -9
done
for o in random few_unique nearly reversed; do
  timeout 120 python tools/profile_one.py --order $o --warmup 5 --flush | grep "last sort" | sed "s/^/$o (no stamps) /"
done
