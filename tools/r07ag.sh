# ncu launch lists + full captures at C4 10 % and C3 (N=1), each after a plain run of the same command
mkdir -p gpurun_out/$1
C4="python bench.py --density 0.1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
C3="python bench.py --rows 800000 --width 1024 --density 0.01 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
KR='k_(bp_begin|extract_tiles|push_scatter|place_tiles2|depth_scan|vacate|fallback|agg_mark|agg_union|agg_values|decode)'
for cfg in C4 C3; do
  CMD=${!cfg}
  timeout 600 $CMD > gpurun_out/$1/short_$cfg.json 2>&1 || continue
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/$1/launches_$cfg.csv $CMD > gpurun_out/$1/ncu_launches_$cfg.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s 30 -c 10 -o gpurun_out/$1/full_$cfg $CMD > gpurun_out/$1/ncu_full_$cfg.log 2>&1
done
