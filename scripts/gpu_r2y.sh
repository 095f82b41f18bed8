# Follow-up: full shared-memory carveout for the persistent kernels. GPU tests, then the C4 sweep at
# 16K and 64K queries (compare ef 224/256 with profiles/r2_bench_C4_batch_sweep.jsonl).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/y_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/y_pytest_gpu.log
for M in 16384 65536; do
  S=$(date +%s)
  timeout 1800 python bench.py --config C4 --m $M --full-sweep --no-full --no-cpu-baseline --no-f1 --entries 32 --steps 5 --warmup 3 \
     --cache /tmp/pa_cache > gpurun_out/y_c4_$M.json 2> gpurun_out/y_c4_$M.log; echo "C4 m=$M rc $? wall $(( $(date +%s) - S ))s"
  python -c "import json;d=json.loads(open('gpurun_out/y_c4_$M.json').read().strip().splitlines()[-1]);print($M, d['value'], d['config']['ef'], d['roofline']['frac'], [(s['ef'], s['recall_at_10'], s['gpu_ms']) for s in d['ef_sweep'] if s['ef']>=160])"
done
