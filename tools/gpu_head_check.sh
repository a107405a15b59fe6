#!/bin/bash
# HEAD check on one B200 (run under gpurun): GPU tests, the bench line and the
# K4 simulator timings in both comm modes.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x > $O/h_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/h_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/h_smoke.log
timeout 900 python bench.py > $O/h_bench.log 2>&1; echo "bench rc=$?"
grep '^{' $O/h_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['parity_vs_reference']['mismatches'])"
for a in "4 seq" "4" "8 seq" "16 seq"; do timeout 300 python tools/sim_bench.py $a >> $O/h_sim.jsonl 2>&1; echo "sim $a rc=$?"; done
tail -4 $O/h_sim.jsonl | cut -c1-300
