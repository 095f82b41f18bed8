# NEXT-f4 (Table 6 ablation on C1) and NEXT-f2 (B200 operating points: sampling -> 1.0, d' -> D,
# GPU-only Recall@10 against the FULL-space ground truth).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --ablation --no-cpu-baseline --variants= --cache /tmp/pa_cache > gpurun_out/bench_ablation.json 2> gpurun_out/bench_ablation.log; echo "ablation rc $?"
python -c "import json;d=json.load(open('gpurun_out/bench_ablation.json'));[print(a['removed'], a['qps_at_0.90'], a['ef']) for a in d['ablation_table6']]"
for SET in "--set ratio=1.0" "--set dp=96" "--set ratio=1.0 --set dp=96" ""; do
  timeout 1500 python bench.py --gt full --no-full --no-cpu-baseline --variants=exact,fp16 --steps 5 $SET --cache /tmp/pa_cache > gpurun_out/bench_f2.json 2> gpurun_out/bench_f2.log
  cat gpurun_out/bench_f2.json >> gpurun_out/bench_f2_all.jsonl
  python -c "import json;d=json.load(open('gpurun_out/bench_f2.json'));print('$SET', d['config']['workload'], d['value'], d['config']['ef'], d['config']['recall_at_10_full_gt_gpu_only'], d['roofline']['traverse_ms'], d['roofline']['frac'], {k:(v['value'],v['ef']) for k,v in d['variants'].items()})"
done
