"""Tensor parallelism over NCCL between processes: two ranks on two GPUs, the communicator
built from a unique id broadcast over a gloo process group, the row-parallel all-reduces and the argmax
max-reduce captured in the decode step's CUDA graph (SF_FLAG_CUDA_GRAPH + a graph-safe collective).
Runs only where >= 2 GPUs are visible (the development box has one); the same model through the
single-GPU local group is covered by test_tensor_parallel_matches_oracle / test_tp_bf16_reduce_parity."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import torch.distributed as dist

    from gpu_helpers import max_seq_for, setup
    from paper_2511_20340_b200 import Engine, EngineConfig
    from paper_2511_20340_b200 import _native as N
    from paper_2511_20340_b200 import tp as tpmod
    from paper_2511_20340_b200.engine import nccl_unique_id
    from synth import get_config

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    cfg = get_config("70b").replace(n_layers=2, d_model=2048, n_heads=16, n_kv_heads=4, d_ff=5632, batch=2,
                                    prompt_len=64, gen_len=8)
    w, prompts = setup(cfg, seed=33, jitter=0.1)
    out = {}
    for fused in (False, True):
        for flags in (0, N.SF_FLAG_CUDA_GRAPH):
            ec = EngineConfig.from_model(cfg, max_batch=2, max_seq=max_seq_for(cfg, 32, cfg.draft_len), tp_size=world,
                                         tp_rank=rank, flags=flags)
            eng = Engine(ec, w)
            eng.attach_nccl(tpmod.share_unique_id(nccl_unique_id, rank), world, rank)
            if fused:  # NEXT-3: the row-parallel all-reduce over peer memory, fused into the consumer
                eng.attach_xch(tpmod.share_xch_handles(eng.xch_handle(), rank, world))
            eng.prefill(prompts.cuda())
            em = torch.zeros(6, 2, cfg.draft_len + 1, dtype=torch.int32, device="cuda")
            eng.decode_steps(6, em, None)
            eng.sync()
            out[(fused, flags)] = em.cpu().numpy().tolist()
            dist.barrier()  # (peers unmap the exchange regions before their owners free them)
            eng.close()
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_tp2_nccl_graph_equals_eager_and_ranks_agree():
    """NCCL all-reduce and the NEXT-3 fused peer-memory all-reduce (CUDA IPC exchange regions)."""
    from paper_2511_20340_b200 import _native as N
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, 29517, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]           # every rank emits the same tokens (NCCL and fused alike)
    for fused in (False, True):       # graph-captured step == eager step
        assert res[0][(fused, 0)] == res[0][(fused, N.SF_FLAG_CUDA_GRAPH)]
