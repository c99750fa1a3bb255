mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests -m gpu -x -q -k "test_dpcg_golden and 2-nd" > gpurun_out/san.log 2>&1; echo "san $?"; grep -v "^$" gpurun_out/san.log | head -60 | cut -c1-250
