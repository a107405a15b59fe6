for m in 2 3 0; do
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA=-DBX_XR_MODE=$m > /dev/null 2>&1
  echo XR=$m; timeout 600 python tools/latency_table.py seq_layered100k_x4 seq_layered100k_x8 seq_wide100k_x16 --no-cpu 2>&1 | cut -c1-120
done
touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc > /dev/null 2>&1
for minb in 2 1; do
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA=-DBX_ROUNDS_MINB=$minb > /dev/null 2>&1
  for bm in 0 120 400; do echo MINB=$minb BIG_MAX=$bm; BX_BIG_MAX=$bm timeout 300 python bench.py --no-cpu-baseline --no-per-graph --steps 3 2>/dev/null | tail -1 | cut -c1-110; done
  echo MINB=$minb single; timeout 300 python tools/latency_table.py layered100k_x4 C1_inception_mtopo_metf --no-cpu 2>&1 | cut -c1-140
done
