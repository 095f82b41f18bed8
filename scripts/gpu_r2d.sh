# Round-2 session D: binary-search rank merge (A/B vs the ballot merge), tests, C3 at 100M.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_d.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu_d.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu_d.log
NB="--no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 --entries 0"
# C2 (100M): generation once into /tmp/pa_cache, then main vs ballot merge, twice each (interleaved)
for rep in 1 2; do
  timeout 1800 python bench.py $NB --ef 224 > gpurun_out/ab_C2_main_$rep.json 2> gpurun_out/ab_C2_main_$rep.log; echo "C2 main rc $?"
  (cd ab/ballot && timeout 900 python bench.py $NB --ef 224 > ../../gpurun_out/ab_C2_ballot_$rep.json 2> ../../gpurun_out/ab_C2_ballot_$rep.log); echo "C2 ballot rc $?"
done
for f in gpurun_out/ab_C2_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
# C1 (10M): main (ballot for SMAX<8) vs bs everywhere
timeout 900 python bench.py --config C1 $NB --ef 80 --cache /tmp/pa_c1 > gpurun_out/ab_C1_main.json 2> gpurun_out/ab_C1_main.log; echo "C1 main rc $?"
(cd ab/bsall && timeout 900 python bench.py --config C1 $NB --ef 80 --cache /tmp/pa_c1 > ../../gpurun_out/ab_C1_bsall.json 2> ../../gpurun_out/ab_C1_bsall.log); echo "C1 bsall rc $?"
for f in gpurun_out/ab_C1_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
# headline operating point with the FES entry-count sweep (GPU stage only)
timeout 900 python bench.py --no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 > gpurun_out/bench_r2d_esweep.json 2> gpurun_out/bench_r2d_esweep.log; echo "esweep rc $?"
grep "E=" gpurun_out/bench_r2d_esweep.log | tail -30
# ncu of the C2 traversal with the new merge
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 4 -c 1 \
   -o gpurun_out/prof_traverse_r2d -f python bench.py --steps 1 --warmup 3 --ef 224 --entries 0 --no-full --no-cpu-baseline --no-f1 > gpurun_out/ncu_full_d.log 2>&1; echo "ncu full rc $?"
# C3 (LAION-shaped 100M x 768, GPU stage)
timeout 2400 python bench.py --config C3 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_C3_r2d.json 2> gpurun_out/bench_C3_r2d.log; echo "C3 rc $?"
tail -4 gpurun_out/bench_C3_r2d.log
