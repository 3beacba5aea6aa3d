cd $GRAFT_REPO_ROOT
timeout 300 python tools/sgd_one.py 1000000000 3 > gpurun_out/sgd_one.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sgd_launches.csv python tools/sgd_one.py 1000000000 3 > gpurun_out/sgd_ncu.log 2>&1
