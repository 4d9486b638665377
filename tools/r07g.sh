mkdir -p gpurun_out/$1
SHORT="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 600 $SHORT > gpurun_out/$1/short.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_agg_fused' -s 3 -c 1 -o gpurun_out/$1/fused1 $SHORT > gpurun_out/$1/ncu.log 2>&1
ZEN_AGG_FUSED=0 timeout 900 ncu --set full --clock-control none -k regex:'k_agg_(mark|union|values)' -s 6 -c 3 -o gpurun_out/$1/legacy1 $SHORT >> gpurun_out/$1/ncu.log 2>&1
