import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2408_14690_b200 import decode as D, engine as E, tp
spec = D.DecoderSpec(1024, 8, 4, 2048, 2, vocab=1024, rope_theta=500000.0, norm_eps=1e-5, max_seq=64)
W = D.random_weights(spec, torch.bfloat16, seed=12)
thr = [[0.3, 0.4, 0.5, 0.02, 0.6, 0.7, 0.05]] * 2
world = 2
ref = E.StepDecoder(W, thr, kv_dtype=torch.float32)
ranks = [tp.TPStepDecoder(tp.shard_weights(W, r, world), thr, rank=r, world=world, kv_dtype=torch.float32) for r in range(world)]
ref.reset(); [d.reset() for d in ranks]
for step, tok in enumerate([5, 17, 999, 3, 250, 7, 7, 42, 11]):
    ref.token.fill_(tok); ref.step_token()
    for d in ranks: d.token.fill_(tok)
    tp.run_lockstep_step(ranks)
    torch.cuda.synchronize()
    fx = lambda a: a.double() / 2**32
    if step in (3, 5):
        for l in range(2):
            for k in ("o", "down"):
                r = fx(ref.acc_views[l][k]); t = fx(ranks[0].dec.acc_views[l][k])
                e = (t - r).abs(); i = int(e.argmax())
                print("  ", l, k, "rel", float((t - r).norm() / r.norm()), "max at", i, float(t[i]), float(r[i]))
            nq, nkv = spec.n_q, spec.n_kv
            r = fx(ref.acc_views[l]["qkv"])
            q = torch.cat([fx(d.dec.acc_views[l]["qkv"])[: nq // world] for d in ranks])
            print("   q rel", float((q - r[:nq]).norm() / r[:nq].norm()))
            gu = torch.cat([fx(d.dec.acc_views[l]["gu"]) for d in ranks])
            print("   ctx rel", float((torch.cat([d.dec.ctx for d in ranks]) - ref.ctx).norm() / ref.ctx.norm()))
        for v in range(5):
            a, b = ranks[0].dec.xv[v], ref.xv[v]
            print("   xv", v, float((a - b).norm() / b.norm()))
    print("step", step, "x rel", float((ranks[0].x - ref.x).norm() / ref.x.norm()), "state", ranks[0].dec.state.tolist(), ref.state.tolist(),
          "tok", int(ranks[0].token.item()), int(ref.token.item()), "kc rel", float((torch.cat([d.dec.kcache[0, :, :3] for d in ranks]) .float() - ref.kcache[0, :, :3].float()).norm() / ref.kcache[0, :, :3].float().norm()))
