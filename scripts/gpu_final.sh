# Round-end style check: smoke, full GPU tests, default bench, torchrun (1 rank) path, reference arm, ncu of the traversal.
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
TAG=${1:-final}
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
fi
timeout 1500 python bench.py --cache /tmp/pa_cache > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc $?"
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print({k:d[k] for k in ('value','ms_per_step','gpu_launches')}, d['roofline']['frac'], d['config']['ef'], d['config']['recall_at_10_gt_sub'], {k:(v['value'],v['ef'],v['traverse_ms']) for k,v in (d.get('variants') or {}).items()}, (d.get('end_to_end_full') or {}).get('value'), d['e2e']['value'], d['cpu_baseline']['value'])"
if [ -z "$SKIP_DIST" ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.log; echo "torchrun rc $?"; cut -c1-300 gpurun_out/bench_torchrun.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 --cache /tmp/pa_cache > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.log; echo "reference rc $?"; cut -c1-300 gpurun_out/bench_reference.json
fi
EF=$(python -c "import json;print(json.load(open('gpurun_out/bench_$TAG.json'))['config']['ef'])" 2>/dev/null || echo 96)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --ef $EF --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/prof_traverse_$TAG -f python bench.py --steps 1 --warmup 3 --ef $EF --no-full --no-cpu-baseline --no-f1 --cache /tmp/pa_cache \
   > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
python scripts/ncu_summary.py gpurun_out/prof_traverse_$TAG.ncu-rep gpurun_out/launches_$TAG.csv > gpurun_out/prof_traverse_$TAG.md 2>&1
grep -E "Duration|dram__bytes|stall samples|Achieved Occ" gpurun_out/prof_traverse_$TAG.md
