# Iteration check: GPU tests (optionally a subset), default bench with the NEXT-f1 variants, and
# extra bench lines given as BENCH_EXTRA="ENV=1 ENV2=2|args1;|args2".
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
TAG=${1:-it}
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -rf -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} --cache /tmp/pa_cache > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc $?"
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['config']['ef'], d['config']['recall_at_10_gt_sub']); [print(k, v['value'], v['ef'], v['traverse_ms'], v['roofline_frac'], v['recall_at_10_gt_sub'], round(v['n_dist_per_q'],1)) for k,v in (d.get('variants') or {}).items()]; print('full', (d.get('end_to_end_full') or {}).get('value'), 'e2e', d['e2e']['value'])"
IFS=';' read -ra EX <<< "$BENCH_EXTRA"
i=0
for a in "${EX[@]}"; do
  i=$((i+1))
  [ -z "$a" ] && continue
  envs="${a%%|*}"; args="${a#*|}"; [ "$envs" = "$a" ] && envs=""
  eval "env $envs timeout 900 python bench.py --steps 5 --warmup 3 --no-full --no-cpu-baseline --variants= --cache /tmp/pa_cache $args" > gpurun_out/bench_${TAG}_x$i.json 2> gpurun_out/bench_${TAG}_x$i.log
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_x$i.json'));print('x$i', '$a', d['value'], d['roofline']['traverse_ms'], d['roofline']['frac'], d['config']['ef'], d['config']['recall_at_10_gt_sub'])"
done
if [ -n "$MINB_EXTRA" ]; then
  PA_TRAV_MINB=$MINB_EXTRA python paper_2503_21206_b200/build.py --force > /dev/null 2>&1
  for a in "" "--bloom 12" "--bloom 11"; do
    timeout 900 python bench.py --steps 5 --warmup 3 --no-full --no-cpu-baseline --variants= $a --cache /tmp/pa_cache > gpurun_out/bench_${TAG}_minb.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_minb.json'));print('minb $MINB_EXTRA', '$a', d['value'], d['roofline']['traverse_ms'], d['roofline']['frac'], d['config']['ef'], d['config']['recall_at_10_gt_sub'])"
  done
  python paper_2503_21206_b200/build.py --force > /dev/null 2>&1
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
     --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-full --no-cpu-baseline --variants= --cache /tmp/pa_cache > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 4 -c 1 \
     -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --ef 96 --no-full --no-cpu-baseline --variants= --cache /tmp/pa_cache > gpurun_out/ncu_full_$TAG.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep gpurun_out/launches_$TAG.csv > gpurun_out/prof_$TAG.md 2>&1
  grep -E "Duration|dram__bytes|stall samples|Achieved Occ|Registers" gpurun_out/prof_$TAG.md; tail -8 gpurun_out/prof_$TAG.md
fi
