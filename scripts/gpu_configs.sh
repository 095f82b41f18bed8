# Measurement on the scaled-size T2I-shaped (IP, D=200, d'=64) and LAION-shaped (D=768, d'=128) configs.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
for C in C2S C3S; do
  timeout 1800 python bench.py --config $C --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.log; echo "$C rc $?"
  grep -E "ef=|FULL|built" gpurun_out/bench_$C.log
  python -c "import json;d=json.load(open('gpurun_out/bench_$C.json'));print('$C', 'qps', d['value'], 'ef', d['config']['ef'], 'recall', d['config']['recall_at_10_gt_sub'], 'roof', d['roofline']['frac'], 'kernels', d['roofline']['kernel_ms'], 'f1', {k:(v['value'],v['ef'],v['traverse_ms']) for k,v in (d.get('variants') or {}).items()}, 'full', (d.get('end_to_end_full') or {}).get('value'), 'cpu', d['cpu_baseline']['value'])"
done
