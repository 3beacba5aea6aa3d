cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 python tools/als_sweep_once.py > gpurun_out/als_once.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'gram_frag_kernel' --launch-skip 3 -c 3 -o gpurun_out/r2s5_gram_o1u3 -f python tools/als_sweep_once.py > gpurun_out/ncu_gram.log 2>&1
