# Round-2 session E/F: GPU tests with the binary-search merge restored; C2 A/B of blocks/SM
# (8 = main, 9, 10: ab/mb*), the FES entry sweep, the tail probe, and ncu of the C2 traversal.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/f_pytest_gpu.log
S=$(date +%s)
timeout 1800 python bench.py --no-full --no-f1 --cache /tmp/pa_cache > gpurun_out/f_bench_C2.json 2> gpurun_out/f_bench_C2.log; echo "bench rc $? wall $(( $(date +%s) - S ))s"
grep "E=" gpurun_out/f_bench_C2.log
NB="--no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 --entries 64 --ef 224 --cache /tmp/pa_cache"
for rep in 1 2; do
  timeout 900 python bench.py $NB > gpurun_out/f_ab_main_$rep.json 2> gpurun_out/f_ab_main_$rep.log; echo "main rc $?"
  for v in mb9 mb10; do
    (cd ab/$v && timeout 900 python bench.py $NB > ../../gpurun_out/f_ab_${v}_$rep.json 2> ../../gpurun_out/f_ab_${v}_$rep.log); echo "$v rc $?"
  done
done
timeout 900 python bench.py $NB --repeat-queries 4 > gpurun_out/f_tail_x4.json 2> gpurun_out/f_tail_x4.log; echo "x4 rc $?"
for f in gpurun_out/f_ab_*.json gpurun_out/f_tail_x4.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/f_launches_C2.csv python bench.py --steps 3 --warmup 3 --ef 224 --entries 64 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/f_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/f_prof_traverse_C2 -f python bench.py --steps 1 --warmup 3 --ef 224 --entries 64 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/f_ncu_full.log 2>&1; echo "ncu full rc $?"
python scripts/ncu_summary.py gpurun_out/f_prof_traverse_C2.ncu-rep gpurun_out/f_launches_C2.csv > gpurun_out/f_prof_traverse_C2.md 2>&1
grep -E "Duration|dram__bytes|stall samples|Achieved Occ" gpurun_out/f_prof_traverse_C2.md
