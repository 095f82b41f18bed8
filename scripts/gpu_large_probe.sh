set -x
cd $GRAFT_REPO_ROOT
export PA_DATAGEN_PROFILE=1 PA_KNN_P=48 PA_KNN_REFINE_PASSES=1
PA_KNN_PART=gen timeout 900 python scripts/large_graph_probe.py C2S > gpurun_out/large_probe_C2S_gen.log 2>&1
PA_KNN_PART=gen PA_CACHE=/tmp/pa_cache timeout 2400 python scripts/large_graph_probe.py C2 > gpurun_out/large_probe_C2_gen.log 2>&1 &
PID=$!
while kill -0 $PID 2>/dev/null; do echo "$(date +%T) $(free -g | awk '/Mem/{print $3}') GB host, $(nvidia-smi --query-gpu=memory.used --format=csv,noheader)" >> gpurun_out/large_probe_C2_mem.log; sleep 15; done
