"""Tensor parallelism (BASELINE config 4).

CPU (gloo, world_size 2): the sharding of tp.shard_weights is checked with the
oracle's arithmetic — column-parallel q/k/v/gate/up shards concatenate to the
full projection, row-parallel o/down partials (each rank thresholding only its
own input channels) all-reduce to the full masked projection, the local masks
concatenate to the global mask.
GPU: the sharded kernels driven in lockstep on one device (tp.run_lockstep,
rank-order fp32 sum = what the all-reduce computes) reproduce the unsharded
decode engine step for step.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import actsparse_ref as R


def _spec():
    from paper_2408_14690_b200.decode import DecoderSpec
    return DecoderSpec(256, 8, 4, 384, 2, vocab=96, rope_theta=10000.0, norm_eps=1e-5, max_seq=16)


def _cpu_weights(spec, seed=0):
    from paper_2408_14690_b200.decode import DecoderWeights, LayerWeights
    g = torch.Generator().manual_seed(seed)
    d, f = spec.d_model, spec.d_ff

    def w(m, n):
        return torch.randn(m, n, generator=g) / m ** 0.5

    layers = [LayerWeights(w(d, spec.n_q + 2 * spec.n_kv), w(spec.n_q, d), w(d, 2 * f), w(f, d),
                           torch.ones(d), torch.ones(d)) for _ in range(spec.n_layers)]
    return DecoderWeights(spec, layers, torch.randn(spec.vocab, d, generator=g), torch.ones(d), w(d, spec.vocab))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_14690_b200 import tp
        spec = _spec()
        W = _cpu_weights(spec)
        S = tp.shard_weights(W, rank, world)
        ls = S.spec
        rng = np.random.default_rng(5)
        h = rng.standard_normal(spec.d_model).astype(np.float32)
        t = 0.6
        lw, sw = W.layers[0], S.layers[0]
        # column-parallel: local q|k|v and gate|up columns of the full product
        full_qkv = R.sparsify(h, t) @ lw.wqkv.numpy()
        loc_qkv = R.sparsify(h, t) @ sw.wqkv.numpy()
        nq, nkv, nql, nkvl = spec.n_q, spec.n_kv, ls.n_q, ls.n_kv
        want = np.concatenate([full_qkv[rank * nql:(rank + 1) * nql],
                               full_qkv[nq + rank * nkvl: nq + (rank + 1) * nkvl],
                               full_qkv[nq + nkv + rank * nkvl: nq + nkv + (rank + 1) * nkvl]])
        ok_col = np.allclose(loc_qkv, want, rtol=1e-5, atol=1e-6)
        # row-parallel: rank-local threshold of its own channels, all-reduce of partials
        ctx = rng.standard_normal(spec.n_q).astype(np.float32)
        loc_ctx = ctx[rank * nql:(rank + 1) * nql]
        part = torch.from_numpy(R.sparsify(loc_ctx, t) @ sw.wo.numpy())
        dist.all_reduce(part)
        full_o = R.sparsify(ctx, t) @ lw.wo.numpy()
        ok_row = np.allclose(part.numpy(), full_o, rtol=1e-5, atol=1e-6)
        inter = rng.standard_normal(spec.d_ff).astype(np.float32)
        fl = ls.d_ff
        part = torch.from_numpy(R.sparsify(inter[rank * fl:(rank + 1) * fl], t) @ sw.wdown.numpy())
        dist.all_reduce(part)
        ok_down = np.allclose(part.numpy(), R.sparsify(inter, t) @ lw.wdown.numpy(), rtol=1e-5, atol=1e-6)
        # the local masks concatenate to the global mask
        bits = torch.from_numpy(R.keep_mask(loc_ctx, t).astype(np.uint8))
        gathered = [torch.empty_like(bits) for _ in range(world)]
        dist.all_gather(gathered, bits)
        ok_mask = np.array_equal(torch.cat(gathered).numpy().astype(bool), R.keep_mask(ctx, t))
        # vocabulary shards of the LM head
        ok_lm = torch.equal(S.lm_head, W.lm_head[:, rank * ls.vocab:(rank + 1) * ls.vocab])
        q.put((rank, ok_col, ok_row, ok_down, ok_mask, ok_lm))
    finally:
        dist.destroy_process_group()


def test_shard_math_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert all(r[1:]), r


def test_shard_spec_validation():
    from paper_2408_14690_b200 import tp
    from paper_2408_14690_b200.decode import LLAMA3_70B
    ls = tp.shard_spec(LLAMA3_70B, 8)
    assert (ls.n_heads, ls.n_kv_heads, ls.d_ff, ls.vocab, ls.head_dim) == (8, 1, 3584, 16032, 128)
    with pytest.raises(ValueError, match="must divide"):
        tp.shard_spec(LLAMA3_70B, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_lockstep_tp_matches_single_gpu(world):
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import tp
    from conftest import rel_err
    spec = D.DecoderSpec(1024, 8, 4, 2816, 2, vocab=1024, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
    W = D.random_weights(spec, torch.bfloat16, seed=11)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = D.SparseDecoder(W, thr)
    ranks = [tp.TPDecoder(tp.shard_weights(W, r, world), thr, rank=r, world=world) for r in range(world)]
    ref.reset()
    for d in ranks:
        d.reset()
    for tok in [5, 17, 999, 3, 250, 7, 7, 42]:
        ref.token.fill_(tok)
        ref.step_token()
        for d in ranks:
            d.token.fill_(tok)
        tp.run_lockstep(ranks)
        torch.cuda.synchronize()
        for d in ranks:
            assert rel_err(d.x.cpu().numpy(), ref.x.cpu().numpy()) < 1e-4
            assert rel_err(d.logits_full.cpu().numpy(), ref.logits.cpu().numpy()) < 1e-3
            assert int(d.token.item()) == int(ref.token.item())


def _tp_spec():
    from paper_2408_14690_b200 import decode as D
    # n_kv = 4 heads x 128: TP 4 leaves one kv head (128 columns) per rank
    return D.DecoderSpec(1024, 8, 4, 2048, 2, vocab=1024, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_step_engine_tp_lockstep_matches_single_gpu(world):
    # persistent step kernel per rank; the row-parallel o/down accumulators
    # are summed (int64, exact) between launches; vocab-parallel argmax.
    # fp32 KV cache: the TP and single-GPU split-K partials differ by ~1e-7
    # (different CTA splits), which a bf16 cache can turn into one-ulp (4e-3)
    # steps of single elements and from there into threshold flips; with an
    # fp32 cache the two agree to ~1e-7 at every step.
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200 import tp
    from conftest import rel_err
    spec = _tp_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=12)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    ranks = [tp.TPStepDecoder(tp.shard_weights(W, r, world), thr, rank=r, world=world, kv_dtype=torch.float32)
             for r in range(world)]
    ref.reset()
    for d in ranks:
        d.reset()
    for tok in [5, 17, 999, 3, 250, 7, 7, 42, 11]:
        ref.token.fill_(tok)
        ref.step_token()
        for d in ranks:
            d.token.fill_(tok)
        tp.run_lockstep_step(ranks)
        torch.cuda.synchronize()
        x0 = ranks[0].x.clone()
        for d in ranks:
            assert torch.equal(d.x, x0)  # replicated residual bit-identical across ranks
            assert int(d.token.item()) == int(ref.token.item())
        assert rel_err(x0.cpu().numpy(), ref.x.cpu().numpy()) < 1e-5


def test_tp_step_shard_shapes_70b():
    # Llama-3-70B at TP 8: 8 q heads + 1 kv head per rank fits the step
    # engine's tiling (n_kv a multiple of 128 columns)
    from paper_2408_14690_b200 import tp
    from paper_2408_14690_b200.decode import LLAMA3_70B
    ls = tp.shard_spec(LLAMA3_70B, 8)
    assert ls.n_q % 256 == 0 and ls.n_kv % 128 == 0 and (ls.n_q + 2 * ls.n_kv) % 256 == 0
    assert ls.d_ff % 128 == 0 and ls.d_model % 256 == 0


def _step_dist_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_14690_b200 import decode as D
        from paper_2408_14690_b200 import engine as E
        from paper_2408_14690_b200 import tp
        torch.cuda.set_device(0)
        spec = _tp_spec()
        W = D.random_weights(spec, torch.bfloat16, seed=12)
        thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
        dec = tp.TPStepDecoder(tp.shard_weights(W, rank, world), thr, rank=rank, world=world,
                               kv_dtype=torch.float32)
        dec.reset()
        xs, toks = [], []
        for tok in [5, 17, 999, 3]:
            dec.token.fill_(tok)
            tp.run_step_dist_step(dec)
            torch.cuda.synchronize()
            xs.append(dec.x.cpu().numpy().copy())
            toks.append(int(dec.token.item()))
        q.put((rank, xs, toks))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_step_engine_tp_torch_distributed_world2():
    # two processes on one GPU (their cooperative launches time-slice), the
    # collectives through torch.distributed (gloo here, NCCL on a multi-GPU box)
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from conftest import rel_err
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=540) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = _tp_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=12)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    ref.reset()
    for i, tok in enumerate([5, 17, 999, 3]):
        ref.token.fill_(tok)
        ref.step_token()
        torch.cuda.synchronize()
        for r in res:
            assert r[2][i] == int(ref.token.item())
            assert rel_err(r[1][i], ref.x.cpu().numpy()) < 1e-5
        assert np.array_equal(res[0][1][i], res[1][1][i])


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_fused_tp_in_kernel_exchange(world):
    # the exchange inside the kernel: ranks' launches run concurrently on one
    # device and add into each other's accumulators / counters
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200 import tp
    from conftest import rel_err
    spec = _tp_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=12)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    grp = tp.FusedTPGroup([tp.shard_weights(W, r, world) for r in range(world)], thr, kv_dtype=torch.float32)
    ref.reset()
    grp.reset()
    for tok in [5, 17, 999, 3, 250, 7]:
        ref.token.fill_(tok)
        ref.step_token()
        grp.set_token(tok)
        grp.step()
        torch.cuda.synchronize()
        x0 = grp.decs[0].x.clone()
        for d in grp.decs:
            assert torch.equal(d.x, x0)
            assert int(d.token.item()) == int(ref.token.item())
        assert rel_err(x0.cpu().numpy(), ref.x.cpu().numpy()) < 1e-5


@pytest.mark.gpu
def test_fused_tp_rank_world1_runs_the_rank_path():
    # FusedTPRank's plumbing (tp table, cooperative launch, epochs, LM ticket
    # on "rank 0") at world 1 against the plain engine
    from paper_2408_14690_b200 import decode as D
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200 import tp
    spec = _tp_spec()
    W = D.random_weights(spec, torch.bfloat16, seed=12)
    thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
    ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
    r0 = tp.FusedTPRank(W, thr, rank=0, world=1, kv_dtype=torch.float32)
    ref.reset()
    r0.reset()
    for tok in [5, 17, 999, 3]:
        ref.token.fill_(tok)
        ref.step_token()
        r0.token.fill_(tok)
        r0.step()
        torch.cuda.synchronize()
        assert int(r0.token.item()) == int(ref.token.item())
        assert torch.equal(r0.x, ref.x)
