# C4-style ef/recall sweep (Recall@10 0.80-0.99) at batch sizes 1K-64K, on the C1 10M index (GPU stage).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
for M in 1000 4000 16000 65536; do
  timeout 1500 python bench.py --m $M --full-sweep --no-full --no-cpu-baseline --variants= --steps 5 > gpurun_out/c4_$M.json 2> gpurun_out/c4_$M.log
  cat gpurun_out/c4_$M.json >> gpurun_out/bench_c4_sweep.jsonl
  python -c "import json;d=json.load(open('gpurun_out/c4_$M.json'));print($M, d['value'], d['config']['ef'], [(s['ef'], s['recall_at_10'], round($M/s['gpu_ms']*1e3)) for s in d['ef_sweep']])"
done
