# Runtime A/B (environment switches) on C1: ENVS="A=1;A=0" x BSETS="--ef 80;..."
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 80 --cache /tmp/pa_cache > /dev/null 2>&1
IFS=';' read -ra E_LIST <<< "$ENVS"
IFS=';' read -ra B_LIST <<< "${BSETS:---ef 80}"
for e in "${E_LIST[@]}"; do for bargs in "${B_LIST[@]}"; do
  eval "env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-full --no-cpu-baseline --variants= ${bargs} --cache /tmp/pa_cache" > gpurun_out/eab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/eab.json'));print('$e | $bargs |', d['value'], 'trav', d['roofline']['traverse_ms'], 'fes', d['roofline']['kernel_ms']['fes'], 'frac', d['roofline']['frac'])"
done; done
