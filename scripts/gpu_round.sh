# One GPU session: tests, smoke, bench, ncu launch list + full capture of the top kernel.
# usage: bash scripts/gpu_round.sh [tag]
TAG=${1:-r1}
mkdir -p gpurun_out
rm -rf /tmp/pa_cache
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/lscpu.txt
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
fi
timeout 1500 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} --cache /tmp/pa_cache > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc $?"
if [ -z "$SKIP_NCU" ]; then
EF=$(python -c "import json;print(json.load(open('gpurun_out/bench_$TAG.json'))['config']['ef'])" 2>/dev/null || echo 32)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --ef $EF --no-full --no-cpu-baseline --cache /tmp/pa_cache \
   > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/prof_traverse_$TAG -f python bench.py --steps 1 --warmup 3 --ef $EF --no-full --no-cpu-baseline --cache /tmp/pa_cache \
   > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
fi
tail -5 gpurun_out/pytest_gpu.log 2>/dev/null; tail -2 gpurun_out/smoke.log 2>/dev/null; tail -25 gpurun_out/bench_$TAG.log
