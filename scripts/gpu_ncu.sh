# ncu --set full of one kernel (regex $1) in the C1 bench at ef $2 (default 96); summary to gpurun_out.
K=${1:-k_fes_select}; EF=${2:-96}; TAG=${3:-x}
mkdir -p gpurun_out; rm -rf /tmp/pa_cache
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --ef $EF --no-full --no-cpu-baseline --cache /tmp/pa_cache $BENCH_EXTRA > gpurun_out/ncu_pre_$TAG.json 2>/dev/null
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
   -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --ef $EF --no-full --no-cpu-baseline --cache /tmp/pa_cache $BENCH_EXTRA \
   > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc $?"
python scripts/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/prof_${TAG}.md 2>&1; head -60 gpurun_out/prof_${TAG}.md
