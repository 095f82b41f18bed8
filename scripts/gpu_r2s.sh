# A/B: k_fes_select min resident blocks (register budget): main = 1 (~120 registers, 4 blocks/SM),
# ab/sel6 (76 registers), ab/sel8 (64 registers); FES parity tests on each; C2 tail probe (40K queries).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in ab/*/paper_2503_21206_b200/libpilotann.so.xz; do xz -d -T8 $f; done
NB="--no-full --no-cpu-baseline --no-f1 --steps 10 --warmup 3 --entries 16 --ef 224 --cache /tmp/pa_cache"
timeout 1800 python bench.py $NB > gpurun_out/s_main_0.json 2> gpurun_out/s_main_0.log; echo "gen+main rc $?"
for rep in 1 2; do
  timeout 900 python bench.py $NB > gpurun_out/s_main_$rep.json 2> gpurun_out/s_main_$rep.log; echo "main rc $?"
  for v in sel6 sel8; do
    (cd ab/$v && timeout 900 python bench.py $NB > ../../gpurun_out/s_${v}_$rep.json 2> ../../gpurun_out/s_${v}_$rep.log); echo "$v rc $?"
  done
done
for f in gpurun_out/s_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],d['config']['ef'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
for v in sel6 sel8; do (cd ab/$v && timeout 600 python -m pytest tests -m gpu -q -x -k "fes or entries or config_parity" > ../../gpurun_out/s_pytest_$v.log 2>&1; echo "$v fes tests rc $?"; tail -1 ../../gpurun_out/s_pytest_$v.log); done
timeout 900 python bench.py $NB --repeat-queries 4 > gpurun_out/s_tail_x4.json 2> gpurun_out/s_tail_x4.log; echo "x4 rc $?"
python -c "import json;d=json.loads(open('gpurun_out/s_tail_x4.json').read().strip().splitlines()[-1]);print('x4',d['value'],d['roofline']['kernel_ms'],d['roofline']['frac'])"
