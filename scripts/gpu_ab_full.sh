# Compile-time A/B of the stages-2-3 GPU kernel: full_gpu QPS at its operating point (C1).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 80 --cache /tmp/pa_cache > /dev/null 2>&1
IFS=';' read -ra AB_LIST <<< "$AB"
for combo in "${AB_LIST[@]}"; do
  eval "env $combo python paper_2503_21206_b200/build.py --force" > /dev/null 2>&1
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --variants= --ef 80 --cache /tmp/pa_cache > gpurun_out/abf.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abf.json'));f=d['full_gpu'];print('$combo |', f['value'], f['ef'], [(s['ef'], s['qps'], s['refine_ms']) for s in f['sweep']])"
done
