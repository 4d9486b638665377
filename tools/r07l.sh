# 2 GPUs: rank-mode timelines of BP and HC (rank 0 and 1)
mkdir -p gpurun_out/$1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/timeline.py --syncs 3 --out gpurun_out/$1/tl_bp_n2.txt > gpurun_out/$1/tl.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/timeline.py --syncs 3 --scheme hc --out gpurun_out/$1/tl_hc_n2.txt >> gpurun_out/$1/tl.log 2>&1
