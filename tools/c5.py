#!/usr/bin/env python3
"""BASELINE config C5: a GPT-2-style step's gradient sync with mixed buckets
(SURVEY.md §8f row f2), one process per GPU (torchrun) or one GPU:

  * sparse bucket: the 50,257 x 1600 token-embedding gradient, row-sparse
    (the batch's tokens), through the BP dense sync (extract -> hash -> push ->
    aggregate -> pull -> decode);
  * top-k bucket: a 16 x 1600^2 block of dense-layer gradient, top-k sparsified
    on the device (zen_sparsify_topk, 1%) and synced through BP's sparse input;
  * dense bucket: the rest of the dense layers, NCCL all-reduce (N > 1);
  * apply: SGD on the embedding with the synced sparse gradient (zen_axpy_sparse).

Times are CUDA events on the launching stream, max over ranks.

  torchrun --nproc-per-node N tools/c5.py [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--vocab", type=int, default=50257)
    ap.add_argument("--dim", type=int, default=1600)
    ap.add_argument("--tokens", type=int, default=8192, help="distinct tokens per step")
    ap.add_argument("--topk", type=float, default=0.01)
    ap.add_argument("--dense-mib", type=int, default=128, help="all-reduce bucket size")
    args = ap.parse_args()
    import numpy as np
    import torch
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_stream(torch.cuda.Stream())
    import paper_2309_13254_b200 as zen
    n = world
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    V, D = args.vocab, args.dim
    emb = torch.zeros(V, D, device="cuda")
    rows = torch.randperm(V, device="cuda", generator=g)[: args.tokens]
    emb[rows] = torch.randn(args.tokens, D, device="cuda", generator=g)
    emb_flat = emb.view(-1)
    lay = torch.randn(16 * D * D, device="cuda", generator=g)  # top-k bucket
    dense = torch.randn(args.dense_mib * (1 << 18), device="cuda", generator=g)  # all-reduce
    param = torch.zeros(V * D, device="cuda")
    m_emb, m_lay = emb_flat.numel(), lay.numel()
    keep = int(np.ceil(args.topk * m_lay))
    bp_emb = zen.BPSynchronizer(n, m_emb, max_nnz=args.tokens * D + 4096,
                                rank=None if n == 1 else rank)
    bp_lay = zen.BPSynchronizer(n, m_lay, max_nnz=keep + 4096, rank=None if n == 1 else rank)
    if n > 1:
        bp_emb.connect_process_group()
        bp_lay.connect_process_group()
    lib, ctx = zen.load(), zen.context()
    import ctypes as C
    ti = torch.empty(keep, dtype=torch.int64, device="cuda")
    tv = torch.empty(keep, dtype=torch.float32, device="cuda")
    got = C.c_uint64()
    stream = torch.cuda.current_stream()

    def step(t):
        t[0].record(stream)
        bp_emb.sync_dense([emb_flat])
        t[1].record(stream)
        ctx.bind_stream()
        assert lib.zen_sparsify_topk(ctx.h, C.c_void_p(lay.data_ptr()), m_lay, args.topk,
                                     C.c_void_p(ti.data_ptr()), C.c_void_p(tv.data_ptr()), keep,
                                     C.byref(got)) == 0
        t[2].record(stream)
        bp_lay.sync_sparse([ti[: got.value]], [tv[: got.value]])
        t[3].record(stream)
        if dist is not None:
            dist.all_reduce(dense)
        t[4].record(stream)
        bp_emb.apply_sgd(param.view(V, D), 0.01)
        t[5].record(stream)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    for _ in range(3):
        step(ev[0])
    torch.cuda.synchronize()
    for k in range(args.steps):
        step(ev[k])
    torch.cuda.synchronize()
    names = ["embedding_bp_sync", "topk_sparsify", "topk_bucket_bp_sync", "dense_allreduce",
             "apply_sgd"]
    per = np.array([[ev[k][i].elapsed_time(ev[k][i + 1]) for i in range(5)]
                    for k in range(args.steps)])
    med = np.median(per, axis=0)
    tot = float(np.median(per.sum(axis=1)))
    if dist is not None:
        t = torch.tensor(list(med) + [tot], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        med, tot = t[:5].cpu().numpy(), float(t[5])
    if rank == 0:
        out = {"config": f"C5 GPT-2-style mixed buckets: embedding {V}x{D} ({args.tokens} tokens), "
                         f"top-k {args.topk:.0%} of a {16 * D * D:,}-element dense block, "
                         f"{args.dense_mib} MiB all-reduce", "n_gpus": world,
               "ms_per_step": round(tot, 4),
               "stage_ms": {k: round(float(v), 4) for k, v in zip(names, med)},
               "data": "synthetic, random-init shapes"}
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
