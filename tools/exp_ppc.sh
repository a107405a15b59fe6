# warp-kernel CTA shape (problems per CTA x resident CTAs per SM) and L1 carveout
run() { for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-per-graph 2>/dev/null | tail -1 | cut -c1-90; done; }
for cfg in "2 6" "1 12" "4 3"; do
  set -- $cfg
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA="-DBX_PPC=$1 -DBX_LIST_MINB=$2" > /dev/null 2>&1
  echo PPC=$1 MINB=$2; run
done
for co in 0 25; do echo "PPC=4 MINB=3 CARVEOUT=$co"; BX_CARVEOUT=$co run; done
