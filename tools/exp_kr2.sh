for kr in 4 8 16; do echo KR=$kr; BX_KR=$kr timeout 600 python tools/latency_table.py layered100k_x8 grid100k_x8 wide100k_x16 C1_inception_mtopo_metf C2_gnmt_metf_coplace --no-cpu 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['case'], d.get('algo'), round(d['gpu_kernel_ms'],2))
    except Exception: pass
"; done
