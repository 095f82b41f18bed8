set -x
cd $GRAFT_REPO_ROOT
export PA_DATAGEN_PROFILE=1 PA_KNN_P=48 PA_KNN_REFINE_PASSES=1
PA_GRAPH_ALPHA=1.0 timeout 1500 python scripts/large_diag.py C2 > gpurun_out/diag_C2_geo_a10.log 2>&1
PA_GRAPH_ALPHA=1.2 timeout 1500 python scripts/large_diag.py C2 > gpurun_out/diag_C2_geo_a12.log 2>&1
