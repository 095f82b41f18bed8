# Probes: tail effect (tiled query batches), reference arm, default bench line.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --cache /tmp/pa_cache > gpurun_out/probe_r1.json 2> gpurun_out/probe_r1.log; echo "r1 rc $?"
for R in 2 4; do
timeout 900 python bench.py --steps 5 --warmup 3 --ef 96 --no-full --no-cpu-baseline --cache /tmp/pa_cache --repeat-queries $R > gpurun_out/probe_r$R.json 2>/dev/null
done
for R in 1 2 4; do python -c "import json;d=json.load(open('gpurun_out/probe_r$R.json'));print('repeat',$R,'qps',d['value'],'kernels',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'])"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 --cache /tmp/pa_cache > gpurun_out/ref.json 2> gpurun_out/ref.log; echo "ref rc $?"; cat gpurun_out/ref.json; tail -3 gpurun_out/ref.log
