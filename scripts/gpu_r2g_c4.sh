# C4 (WIKI-shaped 100M x 768, d'=128, GPU stage): ef/Recall@10 sweep at batch sizes 1K-64K on one B200.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for M in 65536 16384 4096 1024; do
  S=$(date +%s)
  timeout 2400 python bench.py --config C4 --m $M --full-sweep --no-full --no-cpu-baseline --no-f1 --entries 64 --steps 5 --warmup 3 \
     --cache /tmp/pa_cache > gpurun_out/g_c4_$M.json 2> gpurun_out/g_c4_$M.log; echo "C4 m=$M rc $? wall $(( $(date +%s) - S ))s"
  python -c "import json;d=json.load(open('gpurun_out/g_c4_$M.json'));print($M, d['value'], d['config']['ef'], d['roofline']['frac'], [(s['ef'], s['recall_at_10'], round($M/s['gpu_ms']*1e3)) for s in d['ef_sweep']])"
done
grep datagen gpurun_out/g_c4_65536.log | tail -5
