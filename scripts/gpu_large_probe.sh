set -x
cd $GRAFT_REPO_ROOT
export PA_DATAGEN_PROFILE=1
PA_KNN_P=24 PA_KNN_REFINE_PASSES=1 timeout 1200 python scripts/large_graph_probe.py C2S > gpurun_out/large_probe_C2S_p24r1.log 2>&1
PA_KNN_P=48 PA_KNN_REFINE_PASSES=0 timeout 1200 python scripts/large_graph_probe.py C2S > gpurun_out/large_probe_C2S_p48r0.log 2>&1
