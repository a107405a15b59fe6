# single graphs on the warp kernel (now 168 registers, no spills) vs the round kernel
for bm in 1000000000000 0; do echo BX_BIG_MIN=$bm; BX_BIG_MIN=$bm timeout 600 python tools/latency_table.py C1_inception_mtopo_metf C2_gnmt_metf_coplace C3_transformer_msct_tight grid100k_x8 --no-cpu 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['case'], d.get('algo'), round(d['gpu_kernel_ms'],2))
    except Exception: pass
"; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-per-graph 2>/dev/null | tail -1 | cut -c1-90; done
