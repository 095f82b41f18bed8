# C3 (LAION-shaped 100M x 768, d'=128) GPU-stage bench line with the current kernels, then
# C4 (WIKI-shaped 100M x 768) ef/Recall@10 sweep at batch sizes 1K-64K on one B200.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=$(date +%s)
timeout 2700 python bench.py --config C3 --cache /tmp/pa_cache > gpurun_out/g_c3.json 2> gpurun_out/g_c3.log; echo "C3 rc $? wall $(( $(date +%s) - S ))s"
grep "E=\|datagen" gpurun_out/g_c3.log | tail -12
python -c "import json;d=json.loads(open('gpurun_out/g_c3.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['ef'],d['config']['fes_entries'],d['roofline']['kernel_ms'],d['roofline']['frac'],d['e2e']['value'],(d['cpu_baseline'] or {}).get('value'))"
rm -rf /tmp/pa_cache/C3-LAION-100M
for M in 65536 16384 4096 1024; do
  S=$(date +%s)
  timeout 2700 python bench.py --config C4 --m $M --full-sweep --no-full --no-cpu-baseline --no-f1 --entries 32 --steps 5 --warmup 3 \
     --cache /tmp/pa_cache > gpurun_out/g_c4_$M.json 2> gpurun_out/g_c4_$M.log; echo "C4 m=$M rc $? wall $(( $(date +%s) - S ))s"
  python -c "import json;d=json.loads(open('gpurun_out/g_c4_$M.json').read().strip().splitlines()[-1]);print($M, d['value'], d['config']['ef'], d['roofline']['frac'], [(s['ef'], s['recall_at_10'], round($M/s['gpu_ms']*1e3)) for s in d['ef_sweep']])"
done
grep datagen gpurun_out/g_c4_65536.log | tail -8
