# Round-2 session B: tests, C2 headline bench, launch list + ncu captures (traverse, GEMMs), NEXT-f4 experiment.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_b.txt 2>&1
python __graft_entry__.py > gpurun_out/build_b.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_b.log 2>&1; echo "smoke rc $?"
timeout 1200 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu_b.log 2>&1; echo "pytest rc $?"
timeout 2400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.log; echo "bench rc $?"
EF=$(python -c "import json;print(json.loads(open('gpurun_out/bench_r2b.json').read().strip().splitlines()[-1])['config']['ef'])" 2>/dev/null || echo 224)
echo "EF=$EF"
NB="--no-full --no-cpu-baseline --no-f1"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/launches_r2b.csv python bench.py --steps 3 --warmup 3 --ef $EF $NB > gpurun_out/ncu_launch_b.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/prof_traverse_r2b -f python bench.py --steps 1 --warmup 3 --ef $EF $NB > gpurun_out/ncu_full_b.log 2>&1; echo "ncu full rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_project_tc|k_fes_scores_tma|k_fes_select" -s 6 -c 3 \
   -o gpurun_out/prof_gemm_r2b -f python bench.py --steps 1 --warmup 3 --ef $EF $NB > gpurun_out/ncu_gemm_b.log 2>&1; echo "ncu gemm rc $?"
timeout 900 python scripts/f4_fes_vs_twohop.py C3S > gpurun_out/f4_C3S.json 2> gpurun_out/f4_C3S.log; echo "f4 rc $?"
tail -3 gpurun_out/pytest_gpu_b.log; tail -2 gpurun_out/smoke_b.log; tail -5 gpurun_out/bench_r2b.log
