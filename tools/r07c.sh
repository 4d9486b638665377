mkdir -p gpurun_out/$1
bash tools/ab_env.sh $1 ZEN_SIDE_CTAS=64
mv gpurun_out/$1/ab.txt gpurun_out/$1/ab_side64.txt
bash tools/ab_env.sh $1 ZEN_SIDE_CTAS=12
mv gpurun_out/$1/ab.txt gpurun_out/$1/ab_side12.txt
SHORT="python bench.py --density 0.1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 600 $SHORT > gpurun_out/$1/short.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_(push_scatter|place_tiles|depth_scan|agg_mark|agg_union|agg_values|decode)' \
  -s 21 -c 7 -o gpurun_out/$1/full10 $SHORT > gpurun_out/$1/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$1/ncu_full.log
