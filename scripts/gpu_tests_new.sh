cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -x -q -k "strided or stage23 or full_host or ef2_above or candidates_rejects or two_streams" > gpurun_out/tests_new.log 2>&1
tail -5 gpurun_out/tests_new.log
