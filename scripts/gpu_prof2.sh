mkdir -p gpurun_out
export TVB_MV_PLAN=384,24,15,24
python scripts/mv_bench.py 160x80x80 > gpurun_out/prof2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 3 -c 1 -o gpurun_out/matvec_c4_v4 python scripts/mv_bench.py 160x80x80 > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?"
