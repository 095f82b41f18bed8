# C2 (100M) operating-point probe: visited-set sizes x ef, perfect-entry oracle, graph refine passes.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
free -g > gpurun_out/free.txt
PA_DATAGEN_PROFILE=1 timeout 2400 python scripts/c2_probe.py C2 /tmp/pa_cache > gpurun_out/c2_probe_base.log 2>&1; echo "probe base rc $?"
PA_KNN_REFINE_PASSES=2 PROBE_BLOOMS=14,15,0 PA_DATAGEN_PROFILE=1 timeout 2400 python scripts/c2_probe.py C2 /tmp/pa_cache_r2 > gpurun_out/c2_probe_ref2.log 2>&1; echo "probe ref2 rc $?"
tail -40 gpurun_out/c2_probe_base.log; tail -30 gpurun_out/c2_probe_ref2.log
