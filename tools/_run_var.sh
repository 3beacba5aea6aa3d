cd $GRAFT_REPO_ROOT
for v in $VARIANTS; do
  if [ "$v" = "default" ]; then lib=""; else lib="$GRAFT_REPO_ROOT/variants/$v.so"; fi
  echo "== variant '$v'" >> gpurun_out/mvar.log
  CPFIT_LIB=$lib timeout 300 python ${TOOL:-tools/kernel_time.py} ${CASES:-2} >> gpurun_out/mvar.log 2>&1
done
