# whole optimizer runs (north-star loop) at C3 and C4, capped outer iterations
mkdir -p gpurun_out
timeout 900 python scripts/opt_run.py C3 60 > gpurun_out/opt_c3.log 2>&1; echo "C3 $?"; tail -1 gpurun_out/opt_c3.log
timeout 1200 python scripts/opt_run.py C4 60 > gpurun_out/opt_c4.log 2>&1; echo "C4 $?"; tail -1 gpurun_out/opt_c4.log
