mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "fp16 or golden or integer or spill" > gpurun_out/pytest_f16.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_f16.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-full --no-cpu-baseline --cache /tmp/pa_cache --full-sweep > gpurun_out/f32_sweep.json 2> gpurun_out/f32_sweep.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-full --no-cpu-baseline --cache /tmp/pa_cache --full-sweep --reduced fp16 > gpurun_out/f16_sweep.json 2> gpurun_out/f16_sweep.log
grep "ef=" gpurun_out/f16_sweep.log
for f in f32_sweep f16_sweep; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f','ef',d['config']['ef'],'qps',d['value'],'kernels',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'],'recall',d['config']['recall_at_10_gt_sub'])"; done
