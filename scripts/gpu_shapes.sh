# Bench lines on the scaled T2I-shaped (IP, d=200, d'=64) and LAION-shaped (d=768, d'=128) configs.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
for C in C2S C3S; do
  timeout 1800 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.log; echo "$C rc $?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$C.json'));print('$C', d['value'], d['config']['ef'], d['config']['recall_at_10_gt_sub'], d['roofline']['traverse_ms'], d['roofline']['frac'], d['roofline']['kernel_ms'], {k:(v['value'],v['ef']) for k,v in d['variants'].items()}, 'full', (d.get('end_to_end_full') or {}).get('value'), 'full_gpu', (d.get('full_gpu') or {}).get('value'), (d.get('full_gpu') or {}).get('ef'))"
done
