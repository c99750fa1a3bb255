# restriction kernel times (ncu, warm) for rows (16 rows in flight) vs cta, C4
python scripts/prof_solve.py 160 80 80 8 8 > /dev/null 2>&1
for v in rows cta; do
TVB_RESTRICT=$v ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_restrict -s 20 -c 3 --csv python scripts/prof_solve.py 160 80 80 8 8 2>/dev/null | grep -E "duration" | awk -F'","' '{print "'$v'", $NF}'
done
