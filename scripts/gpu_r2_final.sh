# Round-2 end-of-session check on a fresh box: smoke, GPU tests, default bench (C2, cold cache,
# wall-clocked), torchrun 1-rank path, reference arm, launch list + ncu --set full of the traversal.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -rf /tmp/pa_cache
timeout 300 python __graft_entry__.py smoke > gpurun_out/z_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/z_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/z_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/z_pytest_gpu.log
S=$(date +%s)
timeout 1800 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.log; echo "bench rc $? wall $(( $(date +%s) - S ))s"
grep "E=" gpurun_out/z_bench.log
python -c "import json;d=json.loads(open('gpurun_out/z_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['config']['ef'],d['config']['fes_entries'],d['roofline'],d['e2e']['value'],(d['end_to_end_full'] or {}).get('value'),(d['full_gpu'] or {}).get('value'),d['cpu_baseline']['value'],d['clocks'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-full --no-cpu-baseline --no-f1 > gpurun_out/z_bench_torchrun.json 2> gpurun_out/z_bench_torchrun.log; echo "torchrun rc $?"; cut -c1-300 gpurun_out/z_bench_torchrun.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/z_bench_reference.json 2> gpurun_out/z_bench_reference.log; echo "reference rc $?"; cut -c1-300 gpurun_out/z_bench_reference.json
EF=$(python -c "import json;print(json.loads(open('gpurun_out/z_bench.json').read().strip().splitlines()[-1])['config']['ef'])")
E=$(python -c "import json;print(json.loads(open('gpurun_out/z_bench.json').read().strip().splitlines()[-1])['config']['fes_entries'])")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(project|fes|traverse|bucket)" --csv \
   --log-file gpurun_out/z_launches_C2.csv python bench.py --steps 3 --warmup 3 --ef $EF --entries $E --no-full --no-cpu-baseline --no-f1 \
   > gpurun_out/z_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/z_prof_traverse_C2 -f python bench.py --steps 1 --warmup 3 --ef $EF --entries $E --no-full --no-cpu-baseline --no-f1 \
   > gpurun_out/z_ncu_full.log 2>&1; echo "ncu full rc $?"
python scripts/ncu_summary.py gpurun_out/z_prof_traverse_C2.ncu-rep gpurun_out/z_launches_C2.csv > gpurun_out/z_prof_traverse_C2.md 2>&1
grep -E "Duration|dram__bytes|stall samples|Achieved Occ" gpurun_out/z_prof_traverse_C2.md
