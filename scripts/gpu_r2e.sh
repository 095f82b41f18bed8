# Round-2 session E: validation of HEAD (smoke, GPU tests, default bench from a cold cache, wall-clocked).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -rf /tmp/pa_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/e_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/e_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/e_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/e_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/e_pytest_gpu.log
S=$(date +%s)
timeout 1800 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.log; echo "bench rc $? wall $(( $(date +%s) - S ))s"
cut -c1-600 gpurun_out/e_bench.json
S=$(date +%s)
timeout 1800 python bench.py --impl reference > gpurun_out/e_bench_ref.json 2> gpurun_out/e_bench_ref.log; echo "ref rc $? wall $(( $(date +%s) - S ))s"
cut -c1-400 gpurun_out/e_bench_ref.json
