#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, the bench line,
# the latency table, the simulator timing, the ncu launch list of a bench step
# and full captures of the dominant kernels. Outputs in gpurun_out/ev_*.
set -u
O=gpurun_out

timeout 1200 python -m pytest tests -q -m gpu > $O/ev_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/ev_tests.log
timeout 600 python bench.py > $O/ev_bench.log 2>&1; echo "bench rc=$?"
timeout 1500 python tools/latency_table.py layered100k_x4 layered100k_x8 layered100k_x64 grid100k_x8 wide100k_x16 \
  C1_inception_mtopo_metf C1_inception_nocoplace C2_gnmt_metf_coplace C3_transformer_msct_tight \
  seq_layered100k_x4 seq_layered100k_x8 seq_wide100k_x16 > $O/ev_latency.jsonl 2>&1; echo "latency rc=$?"
timeout 400 python tools/latency_table.py c4_layered1M_x64 --no-cpu >> $O/ev_latency.jsonl 2>&1
(timeout 200 python tools/sim_bench.py 4; timeout 200 python tools/sim_bench.py 16) > $O/ev_sim.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ev_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-graph > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_place_list -c 1 -o $O/ev_batch \
  python tools/run_sweep.py > /dev/null 2>&1; echo "ncu batch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_place_rounds -c 1 -o $O/ev_rounds \
  python tools/run_case.py layered100k_x4 > /dev/null 2>&1; echo "ncu rounds rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim_flow -c 1 -o $O/ev_simflow \
  python tools/sim_bench.py 4 > /dev/null 2>&1; echo "ncu sim rc=$?"
ls -la $O | tail -20
