# column-scan loads in flight per lane (BX_SCAN_U) on the big single graphs and the sweep
for u in 8 16 4; do
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA="-DBX_SCAN_U=$u" > /dev/null 2>&1
  echo SCAN_U=$u; timeout 900 python tools/latency_table.py layered100k_x64 layered100k_x8 wide100k_x16 layered100k_x4 --no-cpu 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['case'], round(d['gpu_kernel_ms'],1))
    except Exception: pass
"
  timeout 300 python bench.py --no-cpu-baseline --no-per-graph 2>/dev/null | tail -1 | cut -c1-90
done
