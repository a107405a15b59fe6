# warp-kernel register budget: resident CTAs per SM 7 (72 regs) / 6 / 5 / 8
for mb in ${MINBS:-4 3 2}; do
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA=-DBX_LIST_MINB=$mb > /dev/null 2>&1
  echo LIST_MINB=$mb; for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-per-graph 2>/dev/null | tail -1 | cut -c1-90; done
done
