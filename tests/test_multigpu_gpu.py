"""Multi-GPU tensor parallelism across physical GPUs (BASELINE config 4),
one process per GPU — skipped on boxes with fewer than 2 GPUs (the round's
GPU tests run on one).  The single-GPU harnesses of the same protocols are
test_tp.py (NCCL-variant lockstep, gloo processes, FusedTPGroup).

* NCCL: TPStepDecoder ranks over torch.distributed "nccl" — the rank's step
  kernel split at the row-parallel outputs, an int64 all-reduce between the
  pieces (tp.run_step_dist_step) — against the unsharded engine;
* fused: FusedTPRank ranks exchanging partials and counters over CUDA-IPC
  peer memory inside one persistent launch per token per GPU.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900),
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs")]

TOKENS = [5, 17, 999, 3, 250, 7]


def _spec():
    from paper_2408_14690_b200 import decode as D
    return D.DecoderSpec(1024, 8, 4, 2048, 2, vocab=1024, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2408_14690_b200 import decode as D
        from paper_2408_14690_b200 import tp
        W = D.random_weights(_spec(), torch.bfloat16, seed=12)
        thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
        shard = tp.shard_weights(W, rank, world)
        if mode == "nccl":
            dec = tp.TPStepDecoder(shard, thr, rank=rank, world=world, kv_dtype=torch.float32)
        else:
            dec = tp.FusedTPRank(shard, thr, rank=rank, world=world, kv_dtype=torch.float32)
        dec.reset()
        torch.cuda.synchronize()
        dist.barrier()
        xs, toks = [], []
        for tok in TOKENS:
            dec.token.fill_(tok)
            if mode == "nccl":
                tp.run_step_dist_step(dec)
            else:
                dec.step()
            torch.cuda.synchronize()
            xs.append(dec.x.cpu().numpy().copy())
            toks.append(int(dec.token.item()))
        q.put((rank, xs, toks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["nccl", "fused"])
def test_tp_across_two_gpus_matches_single_gpu(mode):
    from conftest import rel_err
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=800) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = D.random_weights(_spec(), torch.bfloat16, seed=12)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    ref.reset()
    for i, tok in enumerate(TOKENS):
        ref.token.fill_(tok)
        ref.step_token()
        torch.cuda.synchronize()
        for r in res:
            assert r[2][i] == int(ref.token.item())
            assert rel_err(r[1][i], ref.x.cpu().numpy()) < 1e-5
        assert np.array_equal(res[0][1][i], res[1][1][i])  # replicated residual identical on both GPUs
