# round-kernel warps per CTA: 8 (default) vs 4, single-graph cases
for w in 4 8; do
  touch paper_2301_08695_b200/csrc/listsched.cu; make -s -C paper_2301_08695_b200/csrc EXTRA=-DBX_RWARPS=$w > /dev/null 2>&1
  echo RWARPS=$w; timeout 600 python tools/latency_table.py C1_inception_mtopo_metf C2_gnmt_metf_coplace C3_transformer_msct_tight grid100k_x8 wide100k_x16 layered100k_x4 layered100k_x64 --no-cpu 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['case'], d.get('algo'), round(d['gpu_kernel_ms'],2))
    except Exception: pass
"
done
