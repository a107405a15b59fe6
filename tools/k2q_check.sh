#!/bin/bash
# K2q check on one B200 (run under gpurun): parity tests, clock64 phases and
# the layered-chain latency rows vs the reference.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seq_small.py -q -x > $O/q_tests.log 2>&1; echo "k2q tests rc=$?"; tail -3 $O/q_tests.log
timeout 600 python tools/k2s_profile.py seq_refchain100k_x4 seq_refchain100k_x8 > $O/q_prof.jsonl 2>&1; echo "prof rc=$?"; cat $O/q_prof.jsonl
timeout 600 python tools/latency_table.py seq_refchain100k_x4 seq_refchain100k_x8 > $O/q_lat.jsonl 2>&1; echo "lat rc=$?"; cut -c1-300 $O/q_lat.jsonl
