# Resident-kernel phase stamps after a 512 MiB L2 flush (as bench.py), with and
# without the in-kernel code warm-up (SR_NO_WARM=1), per C2 order
mkdir -p gpurun_out/cold
for nw in 0 1; do for o in random few_unique nearly reversed; do
  echo "== $o flush no_warm=$nw"
  if [ $nw = 1 ]; then export SR_NO_WARM=1; else unset SR_NO_WARM; fi
  SR_TIMING=1 timeout 120 python tools/profile_one.py --order $o --warmup 3 --flush > gpurun_out/cold/x.log 2>&1
  grep -E "C splitters|C.route|C.tree|C.end|D.end|E.end|last sort" gpurun_out/cold/x.log | tail -7
done; done
