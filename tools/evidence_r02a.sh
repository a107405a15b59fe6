#!/bin/bash
# Round-2 parity-hole evidence (run under gpurun): compute-sanitizer over every
# kernel, the composite-key clip fallback test, C4 (1M ops x 64 devices) with
# the final kernels bit-exact against the compiled reference in the same run,
# m-SCT at C4, and the reference's layered-chain 100k family.
set -u
O=gpurun_out
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > $O/san_$tool.txt 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 $O/san_$tool.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k composite_key > $O/clip_test.log 2>&1; echo "clip rc=$?"; tail -2 $O/clip_test.log
timeout 1500 python tools/latency_table.py refchain100k_x4 refchain100k_x8 seq_refchain100k_x4 seq_refchain100k_x8 > $O/lat_refchain.jsonl 2>&1; echo "refchain rc=$?"; cut -c1-300 $O/lat_refchain.jsonl
timeout 1500 python tools/latency_table.py c4_layered1M_x64 > $O/lat_c4.jsonl 2>&1; echo "c4 rc=$?"; cut -c1-300 $O/lat_c4.jsonl
timeout 900 python tools/latency_table.py c4_layered1M_x64_sct c4_layered1M_x64_tight --no-cpu >> $O/lat_c4.jsonl 2>&1; echo "c4 sct rc=$?"; tail -2 $O/lat_c4.jsonl | cut -c1-300
