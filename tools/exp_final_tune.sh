run() { for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-per-graph 2>/dev/null | tail -1 | cut -c1-90; done; }
for cfg in "3 4" "4 4" "3 2" "3 8"; do
  set -- $cfg
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA="-DBX_LIST_MINB=$1 -DBX_SCAN_U=$2" > /dev/null 2>&1
  echo LIST_MINB=$1 SCAN_U=$2; run
done
