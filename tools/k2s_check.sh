#!/bin/bash
# K2s check on one B200 (run under gpurun): its parity tests, clock64 phases
# and the layered-chain latency rows vs the reference.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_small_frontier.py tests/test_gpu_seq_small.py -q -x > $O/s_tests.log 2>&1; echo "k2s tests rc=$?"; tail -2 $O/s_tests.log
timeout 600 python tools/k2s_profile.py refchain100k_x4 refchain100k_x8 > $O/s_prof.jsonl 2>&1; echo "prof rc=$?"; cat $O/s_prof.jsonl
timeout 600 python tools/latency_table.py refchain100k_x4 refchain100k_x8 refchain100k_x4_sct > $O/s_lat.jsonl 2>&1; echo "lat rc=$?"; cut -c1-300 $O/s_lat.jsonl
