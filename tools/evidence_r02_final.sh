#!/bin/bash
# Round-2 final evidence on one B200 (run under gpurun): GPU tests, the bench
# line, per-graph latency rows, the LP bench, the ncu launch list of a bench
# step and full captures of the dominant kernels, racecheck.
set -u
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu > $O/fin_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/fin_tests.log
timeout 900 python bench.py > $O/fin_bench.log 2>&1; echo "bench rc=$?"
grep '^{' $O/fin_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['parity_vs_reference'])"
timeout 900 python tools/latency_table.py C1_inception_mtopo_metf C1_inception_nocoplace C2_gnmt_metf_coplace C3_transformer_msct_tight > $O/fin_latency.jsonl 2>&1; echo "latency rc=$?"
timeout 900 python tools/latency_table.py refchain1M_x64 >> $O/fin_latency.jsonl 2>&1; echo "refchain1M rc=$?"; tail -1 $O/fin_latency.jsonl | cut -c1-300
timeout 900 python tools/latency_table.py seq_refchain100k_x4 seq_refchain100k_x8 seq_layered100k_x4 seq_wide100k_x16 >> $O/fin_latency.jsonl 2>&1; echo "seq rc=$?"; tail -4 $O/fin_latency.jsonl | cut -c1-300
timeout 600 python tools/k2s_profile.py seq_refchain100k_x4 refchain100k_x4 > $O/fin_phases.jsonl 2>&1; echo "phases rc=$?"
timeout 900 python tools/lp_bench.py > $O/fin_lp.jsonl 2>&1; echo "lp rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fin_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-graph > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_place_list -c 1 -o $O/fin_batch \
  python tools/run_sweep.py > /dev/null 2>&1; echo "ncu batch rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_place_small -c 1 -o $O/fin_small \
  python tools/run_case.py C1_inception_mtopo_metf > /dev/null 2>&1; echo "ncu small rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_place_seq_small -c 1 -o $O/fin_seqsmall \
  python tools/run_case.py seq_refchain100k_x4 > /dev/null 2>&1; echo "ncu seqsmall rc=$?"
# (compute-sanitizer is closed on this GPU pool: profiles/r02/sanitize_note.txt)
ls -la $O | tail -20
