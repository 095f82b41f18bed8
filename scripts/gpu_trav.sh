# A/B of traversal kernels (PA_TRAVERSE=v1 | pipe) × storage on the C1 instance.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache > /dev/null 2>&1
for T in ${TRAVS:-v1 pipe}; do for R in fp32 fp16; do
  PA_TRAVERSE=$T timeout 600 python bench.py --steps 5 --warmup 3 --ef ${EF:-96} --no-full --no-cpu-baseline --no-f1 --reduced $R --cache /tmp/pa_cache > gpurun_out/trav_${T}_${R}.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/trav_${T}_${R}.json'));print('$T','$R','qps',d['value'],'kernels',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'],'recall',d['config']['recall_at_10_gt_sub'])"
done; done
