mkdir -p gpurun_out/r06e
python tools/timeline.py --syncs 2 --out gpurun_out/r06e/tl_1pct.txt > /dev/null 2>&1
ZEN_DIAG_NOCLAIM=1 python tools/timeline.py --syncs 2 --out gpurun_out/r06e/tl_1pct_noclaim.txt > /dev/null 2>&1
ZEN_DIAG_NOCLAIM=1 python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/r06e/tl_10pct_noclaim.txt > /dev/null 2>&1
python tools/timeline.py --syncs 1 > gpurun_out/r06e/plain.log 2>&1 && ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_push_scatter|k_depth_bp|k_agg_mark|k_decode" -s 8 -c 4 -o gpurun_out/r06e/prof python tools/timeline.py --syncs 1 > gpurun_out/r06e/ncu.log 2>&1
