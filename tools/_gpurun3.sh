cd $GRAFT_REPO_ROOT
timeout 200 python tools/cfg2_step.py 3 > gpurun_out/cfg2_step.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tttp_kernel|mttkrp_kernel' -c 4 -o gpurun_out/r2s5_cfg2 -f python tools/cfg2_step.py 1 > gpurun_out/ncu_cfg2.log 2>&1
