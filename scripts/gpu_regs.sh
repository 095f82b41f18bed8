# Register-budget experiment: traversal built for 6 vs 8 resident blocks/SM.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --cache /tmp/pa_cache > gpurun_out/regs_base.json 2> gpurun_out/regs_base.log
for MINB in 6 8; do
  PA_TRAV_MINB=$MINB python paper_2503_21206_b200/build.py --force > /dev/null 2>&1
  for H in 11 12; do
    PA_HASH_LOG2=$H timeout 600 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --cache /tmp/pa_cache > gpurun_out/regs_${MINB}_${H}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/regs_${MINB}_${H}.json'));print('minb',$MINB,'hash',$H,'qps',d['value'],'kernels',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'])"
  done
done
