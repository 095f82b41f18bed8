# NEXT-f2: Fig 9-style grid of sampling ratio x SVD width on C1 (GPU stage alone, full-space GT).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
for R in 0.33 0.66 1.0; do for DP in 32 48 64 96; do
  timeout 900 python bench.py --gt full --no-full --no-cpu-baseline --variants= --steps 5 --set ratio=$R --set dp=$DP > gpurun_out/f2g.json 2> gpurun_out/f2g.log
  cat gpurun_out/f2g.json >> gpurun_out/bench_f2_grid.jsonl
  python -c "import json;d=json.load(open('gpurun_out/f2g.json'));print('ratio $R dp $DP', d['value'], d['config']['ef'], d['config']['recall_at_10_full_gt_gpu_only'], d['roofline']['traverse_ms'], d['roofline']['frac'])" 2>/dev/null || echo "ratio $R dp $DP failed"
done; done
