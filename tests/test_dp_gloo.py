"""Data-parallel host logic on CPU with a world_size-2 gloo group: batch sharding, max-over-ranks
timing / token-sum aggregation, and that per-rank decoding of a shard reproduces the single-process
result for the same global batch (sequences are independent; no collective on the data path)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2511_20340_b200 import dp
        from synth import get_config, make_prompts, make_weights
        cfg = get_config("tiny").replace(gen_len=10)
        w = make_weights(cfg, seed=0)
        W = O.Weights(cfg, w)
        glob = make_prompts(2 * world, cfg.prompt_len, cfg.vocab)      # global batch, seed 1
        local = dp.shard_rows(glob, rank, world)
        toks = torch.tensor([O.sd_decode(W, row.tolist(), cfg.gen_len)[0] for row in local], dtype=torch.int64)
        allt = dp.gather_rows(toks)
        ms, n = dp.reduce_timing(10.0 * (rank + 1), float(toks.numel()))
        out_q.put((rank, allt.tolist(), ms, n))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_dp_two_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # single-process reference over the same global batch
    import oracle as O
    from synth import get_config, make_prompts, make_weights
    cfg = get_config("tiny").replace(gen_len=10)
    W = O.Weights(cfg, make_weights(cfg, seed=0))
    glob = make_prompts(2 * world, cfg.prompt_len, cfg.vocab)
    ref = [O.sd_decode(W, row.tolist(), cfg.gen_len)[0] for row in glob]
    for rank, allt, ms, n in res:
        assert allt == ref                      # gathered shards == unsharded decode
        assert ms == 10.0 * world               # max over ranks
        assert n == world * 2 * cfg.gen_len     # sum over ranks


def test_shard_rows_validation():
    from paper_2511_20340_b200 import dp
    x = torch.arange(12).reshape(6, 2)
    assert dp.shard_rows(x, 1, 3).tolist() == [[4, 5], [6, 7]]
    with pytest.raises(ValueError):
        dp.shard_rows(x, 0, 4)


def _tp_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20340_b200 import tp as tpmod
        calls = []
        uid = tpmod.share_unique_id(lambda: (calls.append(1), bytes(range(128)))[1], rank)
        lw = tpmod.LazyWeights(lambda n: (calls.append(n), n.upper())[1], ["a", "b"])
        out_q.put((rank, uid, len(calls), lw["b"], sorted(lw), len(lw)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_tp_unique_id_broadcast_gloo():
    """Tensor parallelism plumbing: only rank 0 creates the NCCL unique id; every rank receives the
    same 128 bytes; lazy weights draw a tensor per access."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, uid, ncalls, b, names, n in res:
        assert uid == bytes(range(128))
        assert ncalls == (1 if rank == 0 else 0)  # make_id on rank 0 only (counted before the draw)
        assert b == "B" and names == ["a", "b"] and n == 2


def _xch_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20340_b200 import tp as tpmod
        own = bytes([rank + 1]) * 64
        hs = tpmod.share_xch_handles(own, rank, world)
        bad = None
        try:
            tpmod.share_xch_handles(b"x", rank, world)
        except ValueError as e:
            bad = str(e)
        out_q.put((rank, hs, bad))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_tp_xch_handles_allgather_gloo():
    """NEXT-3 host plumbing: every rank receives all ranks' 64-byte exchange handles in rank order
    (what sf_tp_xch_attach expects); a malformed handle is refused before any collective."""
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_xch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(world)]
    for rank, hs, bad in res:
        assert hs == want
        assert bad and "64 bytes" in bad
