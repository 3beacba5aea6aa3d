cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_drivers.py tests/test_gpu_second_order.py tests/test_gpu_generalized.py tests/test_gpu_dist.py -m gpu -x -q -p no:cacheprovider > gpurun_out/gramtest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gramtest.log
