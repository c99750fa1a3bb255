# run stage costs with alternative builds of the library (scratch_variants/*.so)
cp paper_2203_15115_b200/libtopovox_b200.so /tmp/base.so
for v in scratch_variants/*.so; do
  cp $v paper_2203_15115_b200/libtopovox_b200.so
  echo "$v"; timeout 300 python scripts/stage_cost.py 2>&1 | tail -1
done
cp /tmp/base.so paper_2203_15115_b200/libtopovox_b200.so
echo base; timeout 300 python scripts/stage_cost.py 2>&1 | tail -1
