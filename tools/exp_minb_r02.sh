set -u
for mb in 3 4; do
  rm -rf paper_2301_08695_b200/csrc/_build/listsched.o
  make -s -C paper_2301_08695_b200/csrc -j8 EXTRA="-DBX_LIST_MINB=$mb" > /dev/null 2>&1
  for r in 1 2; do
    timeout 600 python bench.py --no-per-graph --no-cpu-baseline > gpurun_out/b_$mb.log 2>&1
    grep "^{" gpurun_out/b_$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb', $mb, round(d['value']), round(d['pipelining']['serial_value']), round(d['e2e']['value']))"
  done
done
