"""Tensor-parallel TEAL decode (BASELINE config 4: Llama-3-70B over 2/4/8
GPUs of one NVLink/NVSwitch box).  The reference has no
distributed code (SPEC.md:8 puts TP out of its scope); the
split follows the paper's setup and Megatron-style sharding:

* column-parallel — q, k, v (whole heads per rank; GQA: KVH / tp kv heads per
  rank) and gate, up (d_ff / tp columns).  Their input is the replicated
  residual stream, so every rank computes the SAME keep mask locally; no
  communication is needed for masks.
* row-parallel — o (its rank's attention heads' context channels) and down
  (its rank's d_ff intermediate channels).  Their inputs are rank-local, so
  each rank thresholds its own channels: the global mask is the
  concatenation of the local ones, elementwise identical to the single-GPU
  mask.  Each produces a partial d-vector -> ALL-REDUCE(sum) -> residual add
  + sum of squares (``teal_residual_add``).
* LM head: column-parallel over the vocabulary; the per-rank logits are
  all-gathered and every rank takes the same argmax.

So one decode step has 2 all-reduces per layer (d fp32 each) and one
all-gather.  The collectives are pluggable: :func:`run_step_dist` drives
``torch.distributed`` (NCCL over NVLink; stream-ordered), and
:func:`run_lockstep` plays all ranks on one device with an explicit
in-order sum — the same arithmetic (rank-order fp32 sum), used to test the
sharded kernels without a multi-GPU box.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import torch

from . import _clib as C
from . import _runtime as RT
from .decode import DecoderSpec, DecoderWeights, LayerWeights, SparseDecoder


def shard_spec(spec: DecoderSpec, world: int) -> DecoderSpec:
    """Per-rank shape: H/tp q heads, KVH/tp kv heads, d_ff/tp, vocab/tp."""
    if spec.n_heads % world or spec.n_kv_heads % world or spec.d_ff % world or (spec.vocab and spec.vocab % world):
        raise ValueError(f"tensor parallel degree {world} must divide heads {spec.n_heads}, kv heads "
                         f"{spec.n_kv_heads}, d_ff {spec.d_ff} and vocab {spec.vocab}")
    return replace(spec, n_heads=spec.n_heads // world, n_kv_heads=spec.n_kv_heads // world,
                   d_ff=spec.d_ff // world, vocab=spec.vocab // world if spec.vocab else 0,
                   head_dim_=spec.head_dim)


def shard_weights(W: DecoderWeights, rank: int, world: int) -> DecoderWeights:
    """Rank `rank`'s slice of input-major weights (see module docstring)."""
    spec = W.spec
    ls = shard_spec(spec, world)
    nq, nkv, f = spec.n_q, spec.n_kv, spec.d_ff
    nql, nkvl, fl = ls.n_q, ls.n_kv, ls.d_ff
    layers = []
    for lw in W.layers:
        q = lw.wqkv[:, rank * nql:(rank + 1) * nql]
        k = lw.wqkv[:, nq + rank * nkvl: nq + (rank + 1) * nkvl]
        v = lw.wqkv[:, nq + nkv + rank * nkvl: nq + nkv + (rank + 1) * nkvl]
        g = lw.wgu[:, rank * fl:(rank + 1) * fl]
        u = lw.wgu[:, f + rank * fl: f + (rank + 1) * fl]
        layers.append(LayerWeights(
            wqkv=torch.cat([q, k, v], dim=1).contiguous(),
            wo=lw.wo[rank * nql:(rank + 1) * nql].contiguous(),
            wgu=torch.cat([g, u], dim=1).contiguous(),
            wdown=lw.wdown[rank * fl:(rank + 1) * fl].contiguous(),
            rms_attn=lw.rms_attn, rms_mlp=lw.rms_mlp))
    head = None
    if W.lm_head is not None:
        vl = ls.vocab
        head = W.lm_head[:, rank * vl:(rank + 1) * vl].contiguous()
    return DecoderWeights(ls, layers, W.embedding, W.final_norm, head)


class TPDecoder(SparseDecoder):
    """One rank of a tensor-parallel decode.  `weights` are this rank's shard
    (:func:`shard_weights`); thresholds are the model's per-layer lists (the
    same on every rank).  Use :func:`run_step_dist` / :func:`run_lockstep`
    to drive steps; the residual stream ``x`` and the argmax ``token`` end
    up identical on every rank."""

    def __init__(self, weights: DecoderWeights, thresholds=None, rank: int = 0, world: int = 1,
                 full_vocab: int = 0, **kw):
        self.rank, self.world = rank, world
        self.full_vocab = full_vocab or weights.spec.vocab * world
        super().__init__(weights, thresholds, **kw)

    def _build(self, thresholds):
        super()._build(thresholds)
        d = self.spec.d_model
        self.part = torch.zeros(d, device=self.device)
        for (_, o, _, dn) in self.layer_args:
            for a in (o, dn):  # row-parallel: partial projection, reduced across ranks
                a.epilogue = C.EPI_STORE
                a.seg[0].y = self.part.data_ptr()
                a.resid = None
                a.ss_out = None
        if self.lm_args is not None:
            self.logits_full = torch.zeros(self.full_vocab, device=self.device)

    def launches_per_step(self) -> int:
        return 1 + 7 * self.spec.n_layers + (2 if self.lm_args is not None else 0)

    def step_ops(self, stream_h: int, from_token: bool):
        """Generator over one decode step: launches this rank's kernels on
        `stream_h` and yields ('allreduce', tensor) / ('allgather', out, in)
        at every collective point; the driver performs the collective
        (stream-ordered) before resuming."""
        L = C.lib()
        spec = self.spec
        if from_token:
            src, sdt, tok = self.w.embedding.data_ptr(), RT.dtype_code(self.w.embedding.dtype), self.token.data_ptr()
        else:
            src, sdt, tok = self.x_in.data_ptr(), C.TEAL_F32, None
        C.check(L.teal_load_residual(src, sdt, tok, spec.d_model, self.x.data_ptr(), self.ss.data_ptr(),
                                     self.res_tile, self.state.data_ptr(), stream_h))
        len_ptr = self.state.data_ptr() + 4
        for l, (qkv, o, gu, dn) in enumerate(self.layer_args):
            C.check(L.teal_fused_gemv(ctypes.byref(qkv), stream_h))
            C.check(L.teal_decode_attention(self.q.data_ptr(), self.kcache[l].data_ptr(), self.vcache[l].data_ptr(),
                                            RT.dtype_code(self.kv_dtype), spec.n_heads, spec.n_kv_heads,
                                            spec.head_dim, spec.max_seq, len_ptr, spec.max_seq,
                                            self.ctx.data_ptr(), self.ws.data_ptr(), self.tickets.data_ptr(),
                                            self.attn_nsplit, stream_h))
            for args, nxt in ((o, gu), (dn, None)):
                C.check(L.teal_fused_gemv(ctypes.byref(args), stream_h))
                yield ("allreduce", self.part)
                C.check(L.teal_residual_add(self.x.data_ptr(), self.part.data_ptr(), spec.d_model,
                                            self.ss.data_ptr(), self.res_tile, stream_h))
                if nxt is not None:
                    C.check(L.teal_fused_gemv(ctypes.byref(nxt), stream_h))
        if self.lm_args is not None:
            C.check(L.teal_fused_gemv(ctypes.byref(self.lm_args), stream_h))
            yield ("allgather", self.logits_full, self.logits[: spec.vocab])
            C.check(L.teal_argmax(self.logits_full.data_ptr(), self.full_vocab, self.token.data_ptr(),
                                  self.ws.data_ptr(), self.tickets.data_ptr(), stream_h))

    # the single-rank entry points run the generator with an in-place driver
    def _launch_step(self, stream_h: int, from_token: bool) -> None:
        if self.world != 1:
            raise RuntimeError("TPDecoder with world > 1: drive steps with run_step_dist or run_lockstep")
        run_lockstep([self], from_token, stream_h)


def run_step_dist(dec: TPDecoder, from_token: bool = True, group=None) -> None:
    """One step on this rank with torch.distributed collectives (NCCL)."""
    import torch.distributed as dist
    for op in dec.step_ops(RT.stream_handle(), from_token):
        if op[0] == "allreduce":
            dist.all_reduce(op[1], group=group)
        else:
            dist.all_gather_into_tensor(op[1], op[2].contiguous(), group=group)


def run_lockstep(decs, from_token: bool = True, stream_h: int | None = None) -> None:
    """All ranks of a TP group on one device, advanced in lockstep; the
    all-reduce sums the ranks' partials in rank order (fp32) and the
    all-gather concatenates the vocabulary shards."""
    sh = RT.stream_handle() if stream_h is None else stream_h
    gens = [d.step_ops(sh, from_token) for d in decs]
    while True:
        ops = []
        for g in gens:
            try:
                ops.append(next(g))
            except StopIteration:
                ops.append(None)
        if all(o is None for o in ops):
            return
        if any(o is None for o in ops):
            raise RuntimeError("tensor-parallel ranks diverged")
        if ops[0][0] == "allreduce":
            total = ops[0][1].clone()
            for o in ops[1:]:
                total += o[1]
            for o in ops:
                o[1].copy_(total)
        else:
            full = torch.cat([o[2] for o in ops])
            for o in ops:
                o[1].copy_(full)


# ---- tensor parallelism on the persistent step engine ---------------------------
class TPStepDecoder:
    """One rank of a tensor-parallel decode on the persistent step kernel
    (engine.StepDecoder over this rank's weight shard, :func:`shard_weights`).

    The row-parallel o / down projections already reduce their split-K
    partials into int64 fixed-point accumulators (2^-32 units) that the next
    phase's prologue adds to the residual stream.  Tensor parallelism is then
    one integer-sum all-reduce of those accumulators per row-parallel
    projection, between two launches of the step kernel's phase list:

        launch [load, qkv0, attn0, o0]   all-reduce acc_o[0]
        launch [gu0, down0]              all-reduce acc_down[0]
        launch [qkv1, attn1, o1]         all-reduce acc_o[1]  ...
        launch [lm]                      all-gather the per-tile argmax candidates

    Integer addition is exact and associative, so every rank holds the same
    sums whatever the reduction order (NCCL ring / tree / NVLS), and the
    replicated residual stream stays bit-identical across ranks.  Column-
    parallel q/k/v/gate/up masks are computed on the replicated residual
    (identical on every rank); row-parallel masks are rank-local (each rank
    thresholds its own heads' context / its d_ff slice).  Dependencies that
    cross a launch boundary are dropped from the phase list (stream order
    meets them)."""

    def __init__(self, shard: DecoderWeights, thresholds=None, rank: int = 0, world: int = 1,
                 full_vocab: int = 0, **kw):
        from . import engine as E
        self.E = E
        self.rank, self.world = rank, world
        self.dec = E.StepDecoder(shard, thresholds, **kw)
        d = self.dec
        self.spec = d.spec
        self.vocab_local = d.spec.vocab
        self.full_vocab = full_vocab or self.vocab_local * world
        L = d.spec.n_layers
        lm = 1 if d.spec.vocab else 0
        # phase indices: 0 load; layer l: qkv 1+5l, attn 2+5l, o 3+5l, gu 4+5l, down 5+5l; lm 1+5L
        segs = []
        for l in range(L):
            segs.append((0 if l == 0 else 1 + 5 * l, 4 + 5 * l, ("o", l)))
            segs.append((4 + 5 * l, 6 + 5 * l, ("down", l)))
        if lm:
            segs.append((1 + 5 * L, 2 + 5 * L, ("lm", None)))
        self.segments = segs
        # drop cross-launch dependencies (phases and x-ready waits)
        ph, gr = d._phases_host, d._groups_host
        for (b, _, _) in segs:
            if b != 0:
                ph[b].dep_kind = E.DEP_NONE
        for l in range(1, L):
            ph[2 + 5 * l].dep_kind = E.DEP_NONE  # attention: the load ran in the first launch
        for gi in range(len(gr)):
            gr[gi].xwait = -1
        d._upload_plan()
        self.token = d.token
        if lm:
            nt = d.lm_t.ntiles
            self.cand_all_v = torch.empty(world * nt, device=d.device)
            self.cand_all_i = torch.empty(world * nt, device=d.device, dtype=torch.int32)
            self.cand_offs = (torch.arange(world, device=d.device, dtype=torch.int32)
                              .repeat_interleave(nt) * self.vocab_local)

    def reset(self, start_pos: int = 0) -> None:
        self.dec.reset(start_pos)

    @property
    def x(self):
        return self.dec.x

    def step_ops(self, stream_h: int, from_token: bool = True):
        """Generator over one decode step: launches this rank's kernel
        segments on `stream_h` and yields ('allreduce', int64 tensor) /
        ('allgather', out_v, in_v, out_i, in_i) at every collective point."""
        d, C = self.dec, self.E.C
        L = C.lib()
        p = d.plan
        p.emb = d.w.embedding.data_ptr() if from_token else None
        for (b, e, (kind, l)) in self.segments:
            p.phase_begin, p.phase_end = b, e
            C.check(L.teal_step_launch(ctypes.byref(p), stream_h))
            if kind in ("o", "down"):
                yield ("allreduce", d.acc_views[l][kind])
            else:
                yield ("allgather", self.cand_all_v, d.cand_v, self.cand_all_i, d.cand_i)
                self._global_argmax()
        p.phase_begin, p.phase_end = 0, 0

    def _global_argmax(self) -> None:
        # candidates in rank-major order = ascending vocabulary index, so the
        # first maximum is the lowest index among ties (the kernel's rule)
        # (no host synchronisation: the step is CUDA-graph capturable)
        j = torch.argmax(self.cand_all_v).reshape(1)
        self.token.copy_(torch.index_select(self.cand_all_i, 0, j) + torch.index_select(self.cand_offs, 0, j))


def run_step_dist_step(dec: TPStepDecoder, from_token: bool = True, group=None) -> None:
    """One step of a TPStepDecoder rank with torch.distributed collectives:
    NCCL over NVLink (int64 SUM all-reduce of the accumulators, stream-
    ordered), or any other backend through host copies (gloo tests)."""
    import torch.distributed as dist
    nccl = dist.get_backend(group) == "nccl"
    for op in dec.step_ops(RT.stream_handle(), from_token):
        if op[0] == "allreduce":
            if nccl:
                dist.all_reduce(op[1], group=group)
            else:
                h = op[1].cpu()
                dist.all_reduce(h, group=group)
                op[1].copy_(h)
        else:
            for out, inp in ((op[1], op[2]), (op[3], op[4])):
                if nccl:
                    dist.all_gather_into_tensor(out, inp.contiguous(), group=group)
                else:
                    parts = [torch.empty_like(inp, device="cpu") for _ in range(dist.get_world_size(group))]
                    dist.all_gather(parts, inp.cpu(), group=group)
                    out.copy_(torch.cat(parts))


def run_lockstep_step(decs, from_token: bool = True, stream_h: int | None = None) -> None:
    """All ranks of a TPStepDecoder group on one device in lockstep: the
    all-reduce is an int64 sum (exact), the all-gather a concatenation."""
    sh = RT.stream_handle() if stream_h is None else stream_h
    gens = [d.step_ops(sh, from_token) for d in decs]
    while True:
        ops = []
        for g in gens:
            try:
                ops.append(next(g))
            except StopIteration:
                ops.append(None)
        if all(o is None for o in ops):
            return
        if any(o is None for o in ops):
            raise RuntimeError("tensor-parallel ranks diverged")
        if ops[0][0] == "allreduce":
            total = ops[0][1].clone()
            for o in ops[1:]:
                total += o[1]
            for o in ops:
                o[1].copy_(total)
        else:
            vs = torch.cat([o[2] for o in ops])
            is_ = torch.cat([o[4] for o in ops])
            for o in ops:
                o[1].copy_(vs)
                o[3].copy_(is_)


# ---- fused tensor parallelism: the exchange inside the persistent kernel --------
def _attach_tp(d, peers, cand_v, cand_i, lm_ticket, rank: int, world: int, vocab_off: int, noncoop: bool):
    """Point rank `rank`'s StepDecoder `d` at its TP group: the teal_step_tp
    table (every rank's accumulator / counters / epoch / token pointers, the
    LM candidates and ticket on rank 0), row-parallel o/down outputs summed
    into every rank, and every global join counting world ranks' signals."""
    from . import engine as E
    T = E.StepTP()
    for j, pj in enumerate(peers):
        T.acc[j] = pj["acc"].data_ptr()
        T.counters[j] = pj["counters"].data_ptr()
        T.epoch[j] = pj["epoch"].data_ptr()
        T.token[j] = pj["token"].data_ptr()
    T.cand_v, T.cand_i, T.lm_ticket = cand_v.data_ptr(), cand_i.data_ptr(), lm_ticket.data_ptr()
    T.world, T.rank, T.vocab_off = world, rank, vocab_off
    t = torch.frombuffer(bytearray(bytes(T)), dtype=torch.uint8).to(d.device)
    d.plan.tp, d.plan.noncoop = t.data_ptr(), int(noncoop)
    gr, ph = d._groups_host, d._phases_host
    for l in range(d.spec.n_layers):  # row-parallel outputs: o, down
        gr[4 * l + 1].tp_sum = 1
        gr[4 * l + 3].tp_sum = 1
    for p in range(len(ph)):  # global joins now count every rank's signals
        if ph[p].dep_kind == E.DEP_GLOBAL:
            ph[p].target *= world
    gr[2].xwait_target *= world  # gate/up of layer 0 stages x after counter 0
    d._upload_plan()
    return t


class FusedTPGroup:
    """Tensor parallelism with the exchange INSIDE the persistent step kernel:
    one launch per rank per token, no collective calls.  Row-parallel o/down
    contributors add their int64 fixed-point partials straight into every
    rank's accumulator and bump every rank's tile counters (system-scope
    release, `teal_step_tp`); consumers wait for world x CONTRIB per tile, so
    the exchange overlaps the streaming tile by tile.  Step-start zeroing is a
    cross-rank barrier (counter 0 signalled on every rank), a monotonic
    per-rank epoch keeps a fast rank from signalling the next step before a
    slow rank has reset its counters, and the vocabulary-parallel LM head
    reduces its argmax candidates on rank 0 with one cross-rank ticket.

    This class is the single-GPU validation harness of that protocol: every
    rank's shard and buffers live on this device, the ranks' launches run
    concurrently on separate streams (ordinary launches, each with 1/world of
    the resident CTAs) and "peer memory" is the other ranks' buffers.  On a
    multi-GPU box the same tables hold CUDA-IPC-mapped peer pointers."""

    def __init__(self, shards, thresholds=None, **kw):
        from . import engine as E
        self.E = E
        world = len(shards)
        if not 1 <= world <= E.TP_MAX:
            raise ValueError(f"1 <= world <= {E.TP_MAX}")
        E._bind()
        dev = RT.require_cuda()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        code = RT.dtype_code(shards[0].layers[0].wqkv.dtype) if isinstance(shards[0], DecoderWeights) else None
        per_sm = E.C.lib().teal_step_ctas_per_sm(code if code is not None else E.C.TEAL_BF16)
        per = per_sm * sms // world
        self.world = world
        self.decs = [E.StepDecoder(sh, thresholds, ctas=per, **kw) for sh in shards]
        d0 = self.decs[0]
        self.vocab_local = d0.spec.vocab
        nt_lm = d0.lm_t.ntiles if d0.spec.vocab else 0
        self.cand_v = torch.zeros(max(1, world * nt_lm), device=dev)
        self.cand_i = torch.zeros(max(1, world * nt_lm), device=dev, dtype=torch.int32)
        self.lm_ticket = torch.zeros(1, device=dev, dtype=torch.int32)
        self.epochs = [torch.zeros(world, device=dev, dtype=torch.int32) for _ in range(world)]
        self._tp_dev = []
        for r, d in enumerate(self.decs):
            peers = [dict(acc=dj.acc, counters=dj.counters, epoch=self.epochs[j], token=dj.token)
                     for j, dj in enumerate(self.decs)]
            self._tp_dev.append(_attach_tp(d, peers, self.cand_v, self.cand_i, self.lm_ticket, r, world,
                                           r * self.vocab_local, noncoop=True))
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(world)]

    def reset(self, start_pos: int = 0) -> None:
        for d in self.decs:
            d.reset(start_pos)
        for e in self.epochs:
            e.zero_()
        self.lm_ticket.zero_()

    @property
    def token(self):
        return self.decs[0].token

    def set_token(self, tok: int) -> None:
        for d in self.decs:
            d.token.fill_(tok)

    def step(self, from_token: bool = True) -> None:
        """One decode step: every rank's launch, concurrently."""
        cur = torch.cuda.current_stream()
        for st in self.streams:
            st.wait_stream(cur)
        for d, st in zip(self.decs, self.streams):
            d._launch(st.cuda_stream, from_token)
        for st in self.streams:
            cur.wait_stream(st)


class FusedTPRank:
    """One rank (one process, one GPU) of fused tensor parallelism: the same
    in-kernel exchange as :class:`FusedTPGroup`, with the peers' accumulator,
    counter, epoch and token buffers mapped into this process over CUDA IPC
    (torch's tensor IPC; NVLink peer access) once at setup.  Every rank then
    launches its own cooperative step kernel per token — no collective calls
    on the data path.  (On this single-GPU development box only world 1 runs:
    two processes on one GPU time-slice, so their kernels cannot wait for each
    other; the protocol itself is validated by FusedTPGroup.)"""

    def __init__(self, shard, thresholds=None, rank: int = 0, world: int = 1, group=None, **kw):
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        from . import engine as E
        self.rank, self.world = rank, world
        self.dec = d = E.StepDecoder(shard, thresholds, **kw)
        dev = d.device
        self.epoch = torch.zeros(world, device=dev, dtype=torch.int32)
        nt_lm = d.lm_t.ntiles if d.spec.vocab else 0
        mine = dict(acc=d.acc, counters=d.counters, epoch=self.epoch, token=d.token)
        if rank == 0:
            mine.update(cand_v=torch.zeros(max(1, world * nt_lm), device=dev),
                        cand_i=torch.zeros(max(1, world * nt_lm), device=dev, dtype=torch.int32),
                        lm_ticket=torch.zeros(1, device=dev, dtype=torch.int32))
        self._mine = mine
        if world > 1:
            shared = {k: reduce_tensor(v) for k, v in mine.items()}
            allh = [None] * world
            dist.all_gather_object(allh, shared, group=group)
            peers = [mine if j == rank else {k: fn(*args) for k, (fn, args) in h.items()} for j, h in enumerate(allh)]
        else:
            peers = [mine]
        self._peers = peers  # keep the mappings alive
        self._tp_dev = _attach_tp(d, peers, peers[0]["cand_v"], peers[0]["cand_i"], peers[0]["lm_ticket"],
                                  rank, world, rank * d.spec.vocab, noncoop=False)
        self.token = d.token

    def reset(self, start_pos: int = 0) -> None:
        """Call on every rank (then synchronise) before the first step."""
        self.dec.reset(start_pos)
        self.epoch.zero_()
        if self.rank == 0:
            self._mine["lm_ticket"].zero_()

    @property
    def x(self):
        return self.dec.x

    def step(self) -> None:
        self.dec.step_token()
