cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ccd_launches.csv python tools/ccd_profile.py 100480507 4 > gpurun_out/ncu_ccd2.log 2>&1
