"""One rank of a multi-GPU Balanced-Parallelism parity run (launched by
torchrun from tests/test_multi_gpu.py or by hand:

  torchrun --standalone --nproc-per-node 2 tests/mgpu_worker.py [rows] [width] [density]

Each rank is worker+server `rank`; push/pull are NVLink stores into peer
inboxes mapped with CUDA IPC.  Every rank checks its result against the CPU
oracle (bit-exact indices, values and TrafficReport ledger) -- test infra.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    width = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    density = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ngpu = torch.cuda.device_count()
    dev = local % ngpu
    torch.cuda.set_device(dev)
    if world <= ngpu:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:  # oversubscribed (several ranks per GPU, e.g. n = 8 on fewer GPUs):
        # NCCL refuses duplicate GPUs; the handle exchange only needs gloo
        dist.init_process_group("gloo")
    import bench
    import paper_2309_13254_b200 as zen
    from oracle import COracle

    per = int(np.ceil(density * rows))
    m = rows * width
    live = bench.live_rows(rows, per, world, 0.5, 1.05, 3)
    dense = [bench.dense_gradient(rows, width, live[w], 3 + w) for w in range(world)]
    mine = torch.from_numpy(dense[rank]).cuda()
    bp = zen.BPSynchronizer(world, m, max_nnz=per * width + 1024, params=zen.HashParams(seed=5),
                            rank=rank)
    bp.connect_process_group()
    co = COracle()
    want = co.bp_sync(m, [co.to_sparse(d) for d in dense], seed=5)
    ok = True
    side = torch.cuda.Stream()
    for it in range(4):  # eager, then CUDA-graph replays on a side stream
        if it < 2:
            bp.sync_dense([mine])
        else:
            with torch.cuda.stream(side):
                bp.sync_dense([mine])
        bp.wait()
        oi, ov = bp.result()
        gi = oi.cpu().numpy().view(np.uint64)
        gv = ov.cpu().numpy()
        good = np.array_equal(gi, want.idx) and np.array_equal(gv.view(np.uint32),
                                                               want.val.view(np.uint32))
        led, counts, agg = bp.ledger()
        good = good and np.array_equal(led, want.ledger) and np.array_equal(counts, want.counts)
        bal = bp.balance()
        good = good and bal is not None and bal.push_imbalance == want.balance[0] \
            and bal.pull_imbalance == want.balance[1]
        if not good:
            print(f"RANK {rank} iter {it} MISMATCH: {gi.size} vs {want.idx.size}", flush=True)
            ok = False
    st = bp.collision_stats(rank)
    r1, r2 = co.bp_sizes(2.0, 0.1, int(np.count_nonzero(dense[rank])), world)
    wi, wv = co.to_sparse(dense[rank])
    ref = co.hierarchical_hash(m, wi, wv, co.family(5, world, 3, worker=rank), r1, r2)
    if st.serial_writes != ref.serial_writes or st.placed_at_depth != ref.placed_at_depth:
        print(f"RANK {rank} collision stats mismatch", flush=True)
        ok = False
    # Hierarchical Centralization (f3) over the same inputs: NVLink pushes into
    # the partners' IPC arenas + merge-path merge_sum, graph-replayed
    if world & (world - 1) == 0:
        hc = zen.HCSynchronizer(world, m, rank, max_nnz=per * width + 1024)
        hc.connect_process_group()
        wi, wv, led = co.hier_centralization(m, [co.to_sparse(d) for d in dense])
        for it in range(3):
            hc.sync_dense(mine)
            hi, hv = hc.result()
            good = np.array_equal(hi.cpu().numpy().view(np.uint64), wi) and np.array_equal(
                hv.cpu().numpy().view(np.uint32), wv.view(np.uint32))
            sent = [ib + vb for ib, vb in hc.stage_bits()]
            good = good and sent == [int(led[s, 0, rank]) for s in range(led.shape[0])]
            if not good:
                print(f"RANK {rank} HC iter {it} MISMATCH {hi.numel()} vs {wi.size}", flush=True)
                ok = False
        si, sv = co.to_sparse(dense[rank])
        hc.sync_sparse(torch.from_numpy(si.view(np.int64)).cuda(), torch.from_numpy(sv).cuda())
        hi, hv = hc.result()
        if not (np.array_equal(hi.cpu().numpy().view(np.uint64), wi)
                and np.array_equal(hv.cpu().numpy().view(np.uint32), wv.view(np.uint32))):
            print(f"RANK {rank} HC sparse MISMATCH", flush=True)
            ok = False
        del hc
    # runtime scheme choice: HC profiles the first sync, then select_scheme
    auto = zen.AutoSynchronizer(world, m, rank, max_nnz=per * width + 1024)
    auto.connect_process_group()
    agg_i, agg_v = want.idx, want.val
    for it in range(3):
        auto.sync_dense(mine)
        auto.wait()
        ai, av = auto.result()
        if not np.array_equal(ai.cpu().numpy().view(np.uint64), agg_i):
            print(f"RANK {rank} auto iter {it} index MISMATCH ({auto.choice})", flush=True)
            ok = False
    if world & (world - 1) == 0:
        prof = co.profile(m, [[co.to_sparse(d) for d in dense]])
        if auto.profile is None or abs(auto.profile.gamma[world] - prof[1][world]) > 1e-12 \
                or auto.choice != ("balanced-parallelism" if prof[3] == 0
                                   else "hierarchical-centralization"):
            print(f"RANK {rank} auto profile MISMATCH {auto.profile} vs {prof}", flush=True)
            ok = False
    del auto
    # the measured policy: both schemes timed on the device, the faster kept
    auto = zen.AutoSynchronizer(world, m, rank, max_nnz=per * width + 1024, policy="measured")
    auto.connect_process_group()
    for it in range(2):
        auto.sync_dense(mine)
        auto.wait()
        ai, _ = auto.result()
        if not np.array_equal(ai.cpu().numpy().view(np.uint64), want.idx):
            print(f"RANK {rank} auto(measured) iter {it} index MISMATCH", flush=True)
            ok = False
    if world & (world - 1) == 0 and (auto.measured_ms is None or auto.choice not in auto.measured_ms):
        print(f"RANK {rank} auto(measured) no choice {auto.measured_ms}", flush=True)
        ok = False
    del auto
    # the centralized baselines in rank mode (f4): ring centralization and
    # AGsparse point-to-point, same push + fold machinery
    sparse_in = [co.to_sparse(d) for d in dense]
    # OmniReduce-like in rank mode: results per rank, and the sent entries
    om = zen.HCSynchronizer(world, m, rank, max_nnz=per * width + 1024, scheme="omnireduce")
    om.connect_process_group()
    res, led, _ = co.run_scheme("omnireduce", m, sparse_in_all := [co.to_sparse(d) for d in dense])
    rng = (m + world - 1) // world
    mi = sparse_in_all[rank][0]
    slices = [int(np.count_nonzero((mi // rng) == q)) for q in range(world) if q != rank]
    for it in range(2):
        om.sync_dense(mine)
        gi, gv = om.result()
        good = np.array_equal(gi.cpu().numpy().view(np.uint64), res[rank][0]) and \
            np.array_equal(gv.cpu().numpy().view(np.uint32), res[rank][1].view(np.uint32))
        sc = om.sent_counts()
        good = good and sc[:world - 1] == slices and len(set(sc[world - 1:])) == 1
        bal = om.balance(None if world <= ngpu else None)
        _, _, wbal = co.run_scheme("omnireduce", m, sparse_in_all)
        good = good and bal is not None and wbal is not None and \
            (bal.push_imbalance, bal.pull_imbalance) == tuple(wbal)
        if not good:
            print(f"RANK {rank} omnireduce iter {it} MISMATCH {gi.numel()} vs {res[rank][0].size} "
                  f"{sc} {slices}", flush=True)
            ok = False
    del om
    for scheme, name, comm in [("ring", "ring-centralization", None), ("agsparse", "agsparse", None),
                               ("agsparse-ring", "agsparse", "ring"),
                               ("agsparse-hierarchy", "agsparse", "hierarchy")]:
        if scheme != "agsparse" and world & (world - 1):
            continue
        sy = zen.HCSynchronizer(world, m, rank, max_nnz=per * width + 1024, scheme=scheme)
        sy.connect_process_group()
        res, led, _ = co.run_scheme(name, m, sparse_in, comm)
        for it in range(2):
            sy.sync_dense(mine)
            gi, gv = sy.result()
            good = np.array_equal(gi.cpu().numpy().view(np.uint64), res[rank][0]) and \
                np.array_equal(gv.cpu().numpy().view(np.uint32), res[rank][1].view(np.uint32))
            sent = sum(ib + vb for ib, vb in sy.stage_bits())
            good = good and sent == int(led[:, 0, rank].sum())
            if not good:
                print(f"RANK {rank} {scheme} iter {it} MISMATCH {gi.numel()} vs {res[rank][0].size}",
                      flush=True)
                ok = False
        del sy
    # edge cases through sync_sparse: an empty rank, all empty, and values
    # that cancel across ranks (OmniReduce's block decode drops exact zeros)
    rng = np.random.default_rng(99)
    mm = 5000
    base_idx = np.sort(rng.choice(mm, 40, replace=False)).astype(np.uint64)
    cases = {
        "one_empty": [(np.zeros(0, np.uint64), np.zeros(0, np.float32)) if w == 0 else
                      (np.sort(rng.choice(mm, 30, replace=False)).astype(np.uint64),
                       rng.integers(1, 9, 30).astype(np.float32)) for w in range(world)],
        "all_empty": [(np.zeros(0, np.uint64), np.zeros(0, np.float32)) for _ in range(world)],
        "cancel": [(base_idx, np.full(40, 1.0 if w % 2 == 0 else -1.0, np.float32))
                   for w in range(world)],
    }
    for cname, ins in cases.items():
        for scheme, name, comm in [("hc", "sparcml", None), ("ring", "ring-centralization", None),
                                   ("agsparse", "agsparse", None),
                                   ("agsparse-hierarchy", "agsparse", "hierarchy"),
                                   ("omnireduce", "omnireduce", None)]:
            if scheme in ("hc", "ring", "agsparse-hierarchy") and world & (world - 1):
                continue
            sy = zen.HCSynchronizer(world, mm, rank, max_nnz=64, scheme=scheme)
            sy.connect_process_group()
            res, _, _ = co.run_scheme(name, mm, ins, comm)
            i, v = ins[rank]
            sy.sync_sparse(torch.from_numpy(i.view(np.int64)).cuda(), torch.from_numpy(v).cuda())
            gi, gv = sy.result()
            if not (np.array_equal(gi.cpu().numpy().view(np.uint64), res[rank][0]) and
                    np.array_equal(gv.cpu().numpy().view(np.uint32), res[rank][1].view(np.uint32))):
                print(f"RANK {rank} {scheme} {cname} MISMATCH {gi.numel()} vs {res[rank][0].size}",
                      flush=True)
                ok = False
            del sy
    # mixed buckets (f2): the embedding through BP, a dense layer top-k'd on
    # the device then BP, the rest all-reduced over NCCL, one MixedBucketSync
    if world <= ngpu:
        lay_all = [np.random.default_rng(900 + r).standard_normal(50_000).astype(np.float32)
                   for r in range(world)]
        den_all = [np.random.default_rng(700 + r).integers(-8, 9, 20_000).astype(np.float32)
                   for r in range(world)]
        g = [mine, torch.from_numpy(lay_all[rank]).cuda(), torch.from_numpy(den_all[rank]).cuda()]
        mb = zen.MixedBucketSync([("sparse", m), ("topk", 50_000, 0.02), ("dense", 20_000)],
                                 n=world, rank=rank)
        mb.step(g)
        i0, v0 = mb.result(0)
        if not (np.array_equal(i0.cpu().numpy().view(np.uint64), want.idx) and
                np.array_equal(v0.cpu().numpy().view(np.uint32), want.val.view(np.uint32))):
            print(f"RANK {rank} mixed sparse bucket MISMATCH", flush=True)
            ok = False
        tk = [co.sparsify_topk(x, 0.02) for x in lay_all]
        wt = co.bp_sync(50_000, tk)
        i1, v1 = mb.result(1)
        if not (np.array_equal(i1.cpu().numpy().view(np.uint64), wt.idx) and
                np.array_equal(v1.cpu().numpy().view(np.uint32), wt.val.view(np.uint32))):
            print(f"RANK {rank} mixed top-k bucket MISMATCH", flush=True)
            ok = False
        torch.cuda.synchronize()
        if not np.array_equal(g[2].cpu().numpy(), np.sum(den_all, axis=0)):  # integers: exact
            print(f"RANK {rank} mixed dense bucket MISMATCH", flush=True)
            ok = False
        del mb
    flag = torch.tensor([0 if ok else 1], device="cuda" if world <= ngpu else "cpu")
    dist.all_reduce(flag)
    if rank == 0:
        print("MGPU " + ("OK" if int(flag.item()) == 0 else "FAIL") + f" n={world} M={m}", flush=True)
    dist.barrier()
    del bp
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) == 0 else 1)


if __name__ == "__main__":
    main()
