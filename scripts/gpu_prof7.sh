mkdir -p gpurun_out
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_restrict|k_prolong|k_pcg_update|k_coarse_top_rows|k_coarse_bwd|k_coarse_fwd" -s 30 -c 8 -o gpurun_out/c4_defl_full python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu7.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu7.log
