#!/bin/bash
# Sequential-comm fold check on one B200 (run under gpurun): the GPU parity
# suite, then the sequential latency rows vs the reference.
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x > $O/sf_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/sf_tests.log
timeout 900 python tools/latency_table.py seq_wide100k_x16 seq_layered100k_x4 seq_layered100k_x8 > $O/sf_lat.jsonl 2>&1; echo "lat rc=$?"; cut -c1-300 $O/sf_lat.jsonl
