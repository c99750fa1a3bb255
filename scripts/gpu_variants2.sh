cp paper_2203_15115_b200/libtopovox_b200.so /tmp/base.so
for v in scratch_variants/*.so /tmp/base.so; do
  cp $v paper_2203_15115_b200/libtopovox_b200.so
  echo "$v"; timeout 300 python scripts/solve_bench.py C4a 2>&1 | tail -1 | cut -c1-300
done
cp /tmp/base.so paper_2203_15115_b200/libtopovox_b200.so
