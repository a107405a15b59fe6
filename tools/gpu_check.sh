#!/bin/bash
# Iteration check on one B200 (run under gpurun): GPU tests, the bench line,
# the per-graph latency rows the K2s / round kernels are tuned on.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x > $O/chk_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/chk_tests.log
timeout 900 python bench.py > $O/chk_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 $O/chk_bench.log
timeout 1200 python tools/latency_table.py ${LAT_CASES:-C1_inception_mtopo_metf C1_inception_nocoplace C2_gnmt_metf_coplace C3_transformer_msct_tight refchain100k_x4 refchain100k_x8 seq_refchain100k_x4 grid100k_x8} > $O/chk_latency.jsonl 2>&1; echo "latency rc=$?"; cut -c1-260 $O/chk_latency.jsonl
