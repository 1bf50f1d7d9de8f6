import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200.device import get_ctx, to_device_colmajor, dptr
from paper_1905_05107_b200.engine import IsmaEngine
from conftest import make_low_rank
from oracle import isma_oracle as orc
a = make_low_rank(100, 60, 3, np.random.default_rng(7))
ctx = get_ctx()
A = to_device_colmajor(a, ctx.device)
eng = IsmaEngine(ctx, A, k=3, r=9, c=224, criterion="modes", use_graphs=False)
rng = np.random.default_rng(11)
eng.norm_pass()
eng._stage_uniforms(rng)
eng.update_ops(0, eng.S[0].cols(0, 9))
eng.readback(); rec, _ = eng.read_record()
print("rec after bootstrap", rec)
print("sig_upd", eng.sig_upd[:9].cpu().numpy())
G = eng.G.cpu().numpy().reshape(60, 60)
print("G diag[:5]", np.diag(G)[:5], "G rank", np.linalg.matrix_rank(G))
print("Tl[:, :3] norms", np.linalg.norm(eng.Tl.cpu().numpy().reshape(9, 60)[:3], axis=1))
U = eng.S[0].to_numpy(9)
print("U col norms", np.linalg.norm(U, axis=0))
# direct gram_eigh on the same G
sig = torch.empty(60, dtype=torch.float64, device=ctx.device); T = torch.empty(60 * 9, dtype=torch.float64, device=ctx.device)
Gd = torch.as_tensor(np.asfortranarray(G).T.copy().reshape(-1), device=ctx.device)
ctx.gram_eigh(dptr(Gd), 60, 60, 9, sig, dptr(T), 60); print("info", ctx.read_info(3), "sig", sig[:5].cpu().numpy())
print("numpy eig", np.sqrt(np.clip(np.linalg.eigvalsh(G)[::-1][:5], 0, None)))
print("---- full run")
eng2 = IsmaEngine(ctx, A, k=3, r=9, c=224, criterion="modes", use_graphs=False)
orig_fin = eng2.finalize
def fin():
    print("before finalize: l", eng2.l, "sig", eng2.sig[eng2.cur].cpu().numpy())
    U = eng2.S[eng2.cur].to_numpy(9); print("U col norms", np.linalg.norm(U, axis=0))
    v = orig_fin()
    print("after finalize sig", eng2.sig[eng2.cur].cpu().numpy())
    return v
eng2.finalize = fin
tr, v = eng2.run(np.random.default_rng(11), strategy="unf", tau=0.99, finalize=True, keep=3, trace_cls=pod.IterationTrace)
print([ (t.columns_sampled, t.remaining, t.cosines) for t in tr])
o = orc.run(a, 3, c=224, tau=0.99, strategy="unf", seed=11)
print("oracle", o["sigma"], [t["remaining"] for t in o["trace"]])
