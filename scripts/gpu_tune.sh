# Tuning sweep: visited-table layout × hash size × ef on the C1 bench instance (cached within this call).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
TAG=${1:-tune}
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 --no-full --no-cpu-baseline --cache /tmp/pa_cache > gpurun_out/tune_${TAG}_base.json 2> gpurun_out/tune_${TAG}_base.log; echo "base rc $?"
grep -E "ef=|FULL" gpurun_out/tune_${TAG}_base.log
for VIS in ${VISS:-compact wide}; do for EF in ${EFS:-64 96}; do for H in ${HS:-11 12}; do
  PA_VISITED=$VIS PA_HASH_LOG2=$H timeout 600 python bench.py --steps 5 --warmup 3 --ef $EF --no-full --no-cpu-baseline --cache /tmp/pa_cache > gpurun_out/tune_${TAG}_${VIS}_ef${EF}_h${H}.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tune_${TAG}_${VIS}_ef${EF}_h${H}.json'));print('$VIS','ef',$EF,'hash',$H,'qps',d['value'],'kernels',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'],'recall',d['config']['recall_at_10_gt_sub'])"
done; done; done
