cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'solve_reg_kernel' --launch-skip 3 -c 1 -o gpurun_out/r2s5_solve -f python tools/als_sweep_once.py > gpurun_out/ncu_solve.log 2>&1
