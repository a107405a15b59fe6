#!/bin/bash
# Round-2 evidence (run under gpurun): compute-sanitizer (all four tools) over
# every kernel via tools/sanitize_cases.py, then the bench line.
set -u
O=gpurun_out
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > $O/san_$tool.txt 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 $O/san_$tool.txt
done
timeout 1200 python bench.py > $O/ev_bench.log 2>&1; echo "bench rc=$?"
grep '^{' $O/ev_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value']); [print(json.dumps(r)[:260]) for r in d['per_graph'].get('families', [])]"
