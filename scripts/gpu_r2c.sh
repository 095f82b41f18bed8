# Round-2 session C: radix FES select + ef3 ≤ 512: tests, C2 bench, launch list, ncu of the select.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_c.txt 2>&1
python __graft_entry__.py > gpurun_out/build_c.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_c.log 2>&1; echo "smoke rc $?"
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc $?"
timeout 2400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.log; echo "bench rc $?"
EF=$(python -c "import json;print(json.loads(open('gpurun_out/bench_r2c.json').read().strip().splitlines()[-1])['config']['ef'])" 2>/dev/null || echo 224)
NB="--no-full --no-cpu-baseline --no-f1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/launches_r2c.csv python bench.py --steps 3 --warmup 3 --ef $EF $NB > gpurun_out/ncu_launch_c.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fes_select" -s 6 -c 1 \
   -o gpurun_out/prof_select_r2c -f python bench.py --steps 1 --warmup 3 --ef $EF $NB > gpurun_out/ncu_sel_c.log 2>&1; echo "ncu select rc $?"
tail -3 gpurun_out/pytest_gpu_c.log; tail -2 gpurun_out/smoke_c.log; tail -5 gpurun_out/bench_r2c.log
