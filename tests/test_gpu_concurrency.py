"""Concurrent use of the library: dsa_pipeline calls of DIFFERENT configurations
in flight at once on separate streams (and from separate host threads) must
give exactly the results of serial calls -- no hidden global scratch, tensor-map
or table shared between calls (the reference operators are pure and reentrant,
SURVEY threading convention: P/src/trainer.cpp:359-366 calls them from
std::threads)."""
import threading

import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops

pytestmark = pytest.mark.gpu

CFGS = [("c2_vector", {"L": 1024, "keep": 51}, 6), ("c4_threshold", {"L": 1024, "cap": 82}, 5),
        ("c1_bert_base", {"L": 1024, "keep": 51}, 7), ("c3_block", {"L": 1024, "keep": 4}, 3),
        ("c0_smoke", {}, 1)]


def _setup(dev):
    jobs = []
    for name, over, pairs in CFGS:
        p = load_preset(name).replace(batch=pairs, heads=1, **over)
        q, k, v, P = ops.generate(p, npairs=pairs)
        qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
        pipe = ops.Pipeline(p, pairs=pairs, device=dev)
        ref = pipe(qd, kd, vd, Pd).clone()
        torch.cuda.synchronize()
        jobs.append((pipe, qd, kd, vd, Pd, ref))
    return jobs


def test_pipelines_on_concurrent_streams():
    dev = torch.device("cuda:0")
    jobs = _setup(dev)
    streams = [torch.cuda.Stream() for _ in jobs]
    for _ in range(8):
        outs = []
        for (pipe, qd, kd, vd, Pd, _), s in zip(jobs, streams):
            outs.append(pipe(qd, kd, vd, Pd, out=torch.empty_like(qd), stream=s))
        torch.cuda.synchronize()
        for (_, _, _, _, _, ref), z in zip(jobs, outs):
            assert torch.equal(z, ref)


def test_pipelines_from_concurrent_host_threads():
    dev = torch.device("cuda:0")
    jobs = _setup(dev)
    errors = []

    def worker(job):
        try:
            torch.cuda.set_device(dev)
            pipe, qd, kd, vd, Pd, ref = job
            s = torch.cuda.Stream()
            for _ in range(6):
                z = pipe(qd, kd, vd, Pd, out=torch.empty_like(qd), stream=s)
                s.synchronize()
                if not torch.equal(z, ref):
                    errors.append(pipe.p.name)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(j,)) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
