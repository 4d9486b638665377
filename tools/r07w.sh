mkdir -p gpurun_out/$1
export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "single_worker or aggregate_paths or dense_pipeline or edge or fallback or c4 or golden or hash_bitmap" > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
unset ZEN_B200_LIB
bash tools/ab_lib.sh $1
for r in 1 2; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 timeout 200 python bench.py --density 0.1 --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L 10%', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done
unset ZEN_B200_LIB
