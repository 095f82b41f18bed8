# Round-2 session F: GPU tests with 9 blocks/SM + float4-typed row loads; C2 A/B of the
# distance-load variants (ab/nz1 uninitialised predicated loads, ab/nz2 clamped loads,
# ab/pf L2 prefetch of later passes, ab/pg2 two passes in flight, ab/bal wave-balanced grid);
# ncu of the C2 traversal; C1 with 9 vs 8 blocks (ab/c1mb8).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# A/B libraries ship xz-compressed (the snapshot limit is 512 MiB)
for f in ab/*/paper_2503_21206_b200/libpilotann.so.xz; do xz -d -T8 $f; done
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/h_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/h_pytest_gpu.log
S=$(date +%s)
timeout 1800 python bench.py --cache /tmp/pa_cache > gpurun_out/h_bench_C2.json 2> gpurun_out/h_bench_C2.log; echo "bench rc $? wall $(( $(date +%s) - S ))s"
grep "E=" gpurun_out/h_bench_C2.log
python -c "import json;d=json.loads(open('gpurun_out/h_bench_C2.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['ef'],d['config']['fes_entries'],d['roofline']['kernel_ms'],d['roofline']['frac'],d['e2e']['value'],(d['end_to_end_full'] or {}).get('value'),(d['full_gpu'] or {}).get('value'),d['cpu_baseline']['value'])"
NB="--no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 --entries 32 --ef 224 --cache /tmp/pa_cache"
for rep in 1 2; do
  timeout 900 python bench.py $NB > gpurun_out/h_ab_main_$rep.json 2> gpurun_out/h_ab_main_$rep.log; echo "main rc $?"
  for v in nz2 pf bal; do
    (cd ab/$v && timeout 900 python bench.py $NB > ../../gpurun_out/h_ab_${v}_$rep.json 2> ../../gpurun_out/h_ab_${v}_$rep.log); echo "$v rc $?"
  done
done
for f in gpurun_out/h_ab_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/h_prof_traverse_C2 -f python bench.py --steps 1 --warmup 3 --ef 224 --entries 32 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/h_ncu_full.log 2>&1; echo "ncu full rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/h_launches_C2.csv python bench.py --steps 3 --warmup 3 --ef 224 --entries 32 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/h_ncu_launch.log 2>&1; echo "ncu launches rc $?"
python scripts/ncu_summary.py gpurun_out/h_prof_traverse_C2.ncu-rep gpurun_out/h_launches_C2.csv > gpurun_out/h_prof_traverse_C2.md 2>&1
grep -E "Duration|dram__bytes|stall samples|Achieved Occ|Registers" gpurun_out/h_prof_traverse_C2.md
# C1 (10M): 9 blocks (main) vs 8 (ab/c1mb8)
NC="--config C1 --no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 --cache /tmp/pa_c1"
timeout 900 python bench.py $NC > gpurun_out/h_c1_main.json 2> gpurun_out/h_c1_main.log; echo "C1 main rc $?"
(cd ab/c1mb8 && timeout 900 python bench.py $NC > ../../gpurun_out/h_c1_mb8.json 2> ../../gpurun_out/h_c1_mb8.log); echo "C1 mb8 rc $?"
timeout 900 python bench.py $NC > gpurun_out/h_c1_main2.json 2> gpurun_out/h_c1_main2.log; echo "C1 main2 rc $?"
for f in gpurun_out/h_c1_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['config'].get('fes_entries'),d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
