# A/B of traversal tuning constants at C2 (needs the C2 cache in /tmp/pa_cache from an earlier call on
# this box, else it is rebuilt once).  Variants are built in scratch copies (scripts/ab_variant.sh).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_ab.log 2>&1
declare -A V
V[base]=""
V[deep2]="-DPA_TRAV_MINB_BLOOM=6 -DPA_DIST_PG_MUL=2"
V[l8]="-DPA_GROUP_L32=8"
V[l8deep]="-DPA_GROUP_L32=8 -DPA_TRAV_MINB_BLOOM=6 -DPA_DIST_PG_MUL=2"
V[minb7]="-DPA_TRAV_MINB_BLOOM=7 -DPA_DIST_PG_MUL=2"
for t in deep2 l8 l8deep minb7; do
  bash scripts/ab_variant.sh $t "${V[$t]}" > gpurun_out/ab_build_$t.log 2>&1 &
done
wait
for t in base deep2 l8 l8deep minb7; do
  D=/tmp/ab_$t; [ $t = base ] && D=$GRAFT_REPO_ROOT
  (cd $D && PROBE_BLOOMS=13 PROBE_EFS=160,224 PROBE_ORACLE=0 PA_DATAGEN_QUIET=1 timeout 1800 python scripts/c2_probe.py C2 /tmp/pa_cache) > gpurun_out/ab_$t.log 2>&1
  echo "== $t ${V[$t]}"; grep GPU gpurun_out/ab_$t.log
done
