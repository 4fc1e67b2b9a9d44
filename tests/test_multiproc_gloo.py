"""The N > 1 host path on CPU: world_size 2 over gloo (127.0.0.1).

Ranks own contiguous (b,h)-pair ranges with no collective on the hot path;
after "timing" the per-pair checksums are all-gathered and Z blocks are
gathered to rank 0 by point-to-point sends.  The CPU stand-in for the GPU
work is the oracle's sparse attention on each rank's pairs, so the gathered
result must equal a single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_11299_b200.shard import (gather_checksums, gather_to_rank0, pair_checksums,
                                         pair_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_pair_range_partitions_exactly():
    for pairs in (1, 5, 96, 128, 512):
        for world in (1, 2, 3, 4, 8):
            spans = [pair_range(r, world, pairs) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == pairs
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    # BASELINE configs divide evenly over 1/2/4/8 GPUs
    for pairs in (96, 128, 64, 512):
        for world in (1, 2, 4, 8):
            assert len({b - a for a, b in (pair_range(r, world, pairs) for r in range(world))}) == 1


def _work(pair_ids, L=48, d=16, keep=6):
    from oracle.oracle import Oracle
    o = Oracle()
    zs, nnz = [], []
    for pid in pair_ids:
        rng = np.random.default_rng(1000 + pid)
        q, k, v = rng.normal(size=(3, L, d))
        cols = np.concatenate([np.sort(rng.choice(L, keep, replace=False)) for _ in range(L)]).astype(np.uint32)
        rp = np.arange(0, L * keep + 1, keep, dtype=np.uint64)
        z, _ = o.sparse_attention(q, k, v, rp, cols)
        zs.append(z)
        nnz.append(L * keep)
    return torch.tensor(np.stack(zs)), torch.tensor(nnz, dtype=torch.float64)


def _worker(rank, world, port, pairs, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = pair_range(rank, world, pairs)
    z, nnz = _work(range(lo, hi))
    cs = gather_checksums(pair_checksums(z, nnz), pairs)
    full = gather_to_rank0(z, pairs)
    if rank == 0:
        torch.save({"cs": cs, "z": full}, out)
    dist.barrier()
    dist.destroy_process_group()


def _bench_stub_pairs(p, q, k, v, P):
    """CPU stand-in for dsa_pipeline on a rank's pairs: the oracle's O1 -> O4
    -> O7 chain (the GPU path is pinned to it by the -m gpu parity tests)."""
    from oracle.oracle import Oracle
    o = Oracle()
    Pn = P.double().numpy()
    zs = []
    for i in range(q.shape[0]):
        qn, kn, vn = (t[i].double().numpy() for t in (q, k, v))
        lq, _ = o.levels(qn, Pn, p.bits)
        lk, _ = o.levels(kn, Pn, p.bits)
        m = o.mask_colvec(lq, lk, p.vec_v, p.keep)
        rows = [m[r // p.vec_v] for r in range(p.L)]
        rp = np.arange(0, p.L * p.keep + 1, p.keep, dtype=np.uint64)
        z, _ = o.sparse_attention(qn, kn, vn, rp, np.concatenate(rows), True, False)
        zs.append(z)
    return torch.tensor(np.stack(zs)) if zs else torch.zeros((0, p.L, p.d), dtype=torch.float64)


def _bench_preset():
    from paper_2110_11299_b200 import load_preset
    return load_preset("c2_vector").replace(batch=5, heads=1, L=256, keep=13)


def _bench_worker(rank, world, port, out):
    """bench.py's own rank code (rank_slice / rank_inputs / global_checksum)
    with the CPU stub in place of the GPU pipeline."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    p = _bench_preset()
    lo, hi, q, k, v, P = bench.rank_inputs(p, rank, world)
    assert (lo, hi) == bench.rank_slice(p, rank, world)
    z = _bench_stub_pairs(p, q, k, v, P)
    cs = bench.global_checksum(z, p, world)
    full = gather_to_rank0(z, p.pairs)
    if rank == 0:
        torch.save({"cs": cs, "z": full, "slices": [bench.rank_slice(p, r, world) for r in range(world)]}, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_bench_rank_partition_world2_matches_world1(tmp_path):
    """Strong scaling as bench.py runs it: the config's pairs split over two
    gloo ranks (5 pairs -> 3 + 2), per-pair checksums all-gathered; the
    checksum and Z equal the single-rank run's."""
    import bench
    out = str(tmp_path / "bench.pt")
    mp.spawn(_bench_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = torch.load(out)
    p = _bench_preset()
    assert res["slices"] == [(0, 3), (3, 5)]
    lo, hi, q, k, v, P = bench.rank_inputs(p, 0, 1)
    assert (lo, hi) == (0, 5)
    z1 = _bench_stub_pairs(p, q, k, v, P)
    assert torch.equal(res["z"], z1)
    assert res["cs"] == bench.global_checksum(z1, p, 1)


@pytest.mark.timeout(300)
def test_gloo_world2_matches_single_process(tmp_path):
    pairs = 6
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), pairs, out), nprocs=2, join=True)
    res = torch.load(out)
    z1, nnz1 = _work(range(pairs))
    assert torch.equal(res["z"], z1)
    assert torch.equal(res["cs"], pair_checksums(z1, nnz1))
