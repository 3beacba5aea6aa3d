cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ingest.py tests/test_gpu_hypersparse.py tests/test_gpu_drivers.py -m gpu -x -q -p no:cacheprovider > gpurun_out/sorttest.log 2>&1; echo "pytest exit $?" >> gpurun_out/sorttest.log
for v in default rs8 rs9; do
  if [ "$v" = "default" ]; then lib=""; else lib="$GRAFT_REPO_ROOT/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/sortbench.log
  CPFIT_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-als --no-dense --no-cpu-baseline --no-cpu-ref > gpurun_out/sortbench_$v.json 2>> gpurun_out/sortbench.log
done
