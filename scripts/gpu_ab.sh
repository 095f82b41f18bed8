# Compile-time A/B: rebuild with each env combo in AB="A=1 B=0;A=0 B=1" and bench it (C1, fixed ef).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
TAG=${1:-ab}
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 96 --cache /tmp/pa_cache > /dev/null 2>&1
IFS=';' read -ra AB_LIST <<< "$AB"
for combo in "${AB_LIST[@]}"; do
  eval "env $combo python paper_2503_21206_b200/build.py --force" > /dev/null 2>&1
  for a in ${BARGS:-"--ef 96"}; do :; done
  eval "timeout 600 python bench.py --steps 10 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 96 ${BARGS} --cache /tmp/pa_cache" > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$combo', d['value'], 'trav', d['roofline']['traverse_ms'], 'fes', d['roofline']['kernel_ms']['fes'], 'frac', d['roofline']['frac'])"
  eval "timeout 600 python bench.py --steps 10 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 96 --reduced fp16 ${BARGS} --cache /tmp/pa_cache" > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$combo fp16', d['value'], 'trav', d['roofline']['traverse_ms'], 'fes', d['roofline']['kernel_ms']['fes'], 'frac', d['roofline']['frac'])"
done
