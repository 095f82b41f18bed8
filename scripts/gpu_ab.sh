# Compile-time A/B: rebuild with each env combo in AB="A=1 B=0;A=0 B=1" and bench every
# argument set in BSETS="--ef 96;--ef 96 --bloom 12" (C1 unless --config is given).
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
TAG=${1:-ab}
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-full --no-cpu-baseline --variants= --ef 96 --cache /tmp/pa_cache > /dev/null 2>&1
IFS=';' read -ra AB_LIST <<< "$AB"
IFS=';' read -ra B_LIST <<< "${BSETS:---ef 96;--ef 96 --reduced fp16}"
for combo in "${AB_LIST[@]}"; do
  eval "env $combo python paper_2503_21206_b200/build.py --force" > /dev/null 2>&1
  for bargs in "${B_LIST[@]}"; do
    eval "timeout 600 python bench.py --steps 10 --warmup 3 --no-full --no-cpu-baseline --variants= ${bargs} --cache /tmp/pa_cache" > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$combo | $bargs |', d['value'], 'trav', d['roofline']['traverse_ms'], 'fes', d['roofline']['kernel_ms']['fes'], 'frac', d['roofline']['frac'])"
  done
done
