# Occupancy experiment for the pipelined traversal: register budget (MINB) × hash size × storage.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --ef 96 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache > /dev/null 2>&1
for MINB in 6 8; do
  PA_TRAV_MINB=$MINB python paper_2503_21206_b200/build.py --force > /dev/null 2>&1
  for R in fp32 fp16; do for H in 11 12; do
    PA_HASH_LOG2=$H timeout 600 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --no-f1 --reduced $R --cache /tmp/pa_cache > gpurun_out/occ_${MINB}_${R}_${H}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/occ_${MINB}_${R}_${H}.json'));print('minb',$MINB,'$R','hash',$H,'qps',d['value'],'trav',d['roofline']['traverse_ms'],'frac',d['roofline']['frac'])"
  done; done
done
