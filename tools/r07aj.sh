mkdir -p gpurun_out/$1
export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wire.py -x -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
unset ZEN_B200_LIB
for r in 1 2 3; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 for d in 0.01 0.1; do
 timeout 200 python bench.py --density $d --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L dens=$d', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done; done
unset ZEN_B200_LIB
