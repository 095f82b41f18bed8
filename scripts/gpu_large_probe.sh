set -x
cd $GRAFT_REPO_ROOT
export PA_DATAGEN_PROFILE=1 PA_KNN_P=48 PA_KNN_REFINE_PASSES=1 PA_GRAPH_ALPHA=1.0
PA_GRAPH_FILL=1 PA_CACHE=/tmp/pa_cache timeout 1500 python scripts/large_diag.py C2 > gpurun_out/diag_C2_fill.log 2>&1
PA_GRAPH_FILL=0 DIAG_ORACLE=0 PA_CACHE=/tmp/pa_cache_nofill timeout 1500 python scripts/large_diag.py C2 > gpurun_out/diag_C2_nofill.log 2>&1
