mkdir -p gpurun_out/$1
bash tools/ab_env.sh $1 ZEN_SIDE_TAIL_PRIO=1
mv gpurun_out/$1/ab.txt gpurun_out/$1/ab_tail.txt
ZEN_SIDE_TAIL_PRIO=1 python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_tail.txt > /dev/null 2>&1
for r in 1 2; do for U in 0 1; do
 ZEN_SIDE_TAIL_PRIO=1 ZEN_UNION_ENTRIES=$U timeout 200 python bench.py --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tail=1 entries=$U n1', d['value'])" >> gpurun_out/$1/ab_combo.txt
done; done
