mkdir -p gpurun_out/$1
for r in 1 2; do for N in 2 4; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$r$N$([ $L = ab ] && echo 1 || echo 0) bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep -v NCCL | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L N=$N', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done; done
for r in 1 2; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 timeout 200 python bench.py --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L N=1', d['value'])" >> gpurun_out/$1/ab.txt
done; done
unset ZEN_B200_LIB
