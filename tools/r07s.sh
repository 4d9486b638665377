mkdir -p gpurun_out/$1
bash tools/ab_env.sh $1 ZEN_SIDE_PDL=1
mv gpurun_out/$1/ab.txt gpurun_out/$1/ab_pdl.txt
bash tools/ab_env.sh $1 ZEN_SIDE_PRIO=0
mv gpurun_out/$1/ab.txt gpurun_out/$1/ab_prio.txt
ZEN_SIDE_PDL=1 python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_pdl.txt > /dev/null 2>&1
