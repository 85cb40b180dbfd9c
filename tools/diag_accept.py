import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import oracle, qmcgen
import paper_1708_02645_b200 as q
dev = torch.device("cuda:0")
cfg = qmcgen.CONFIGS["C2"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
R, k, rt, _ = qmcgen.host_instance(cfg, walkers=np.arange(32))
fn = qmcgen.make_functor(cfg.seed, cfg.L, m)
print("m =", m)
S = np.random.default_rng(0).normal(size=(32, 5, R.shape[2])).astype(np.float32)
acc = np.ones(32, np.int32)
Rd, Sd = torch.from_numpy(R).to(dev), torch.from_numpy(S).to(dev)
kd, td = torch.from_numpy(k).to(dev), torch.from_numpy(rt).to(dev)
out = q.eval(Rd, kd, td, fn, cfg.N, cfg.n_up)
q.accept(Rd, Sd, kd, td, torch.from_numpy(acc).to(dev), out, fn, cfg.N, cfg.n_up)
R2, S2, ab = oracle.accept(R, S, k, rt[:, 0], acc, fn, cfg.N, cfg.n_up)
Sg = Sd.cpu().numpy()[:, :, :cfg.N]
err = oracle.normalized_error_state(Sg, S2[:, :, :cfg.N], ab[:, :, :cfg.N], fn)
for c in range(5):
    e = err[:, c]
    w, i = np.unravel_index(np.argmax(e), e.shape)
    print(c, e.max(), "w", w, "i", i, "k", k[w], "gpu", Sg[w, c, i], "orc", S2[w, c, i], "abs", ab[w, c, i], "old", S[w, c, i])
# also k entries only
ek = np.array([err[w, :, k[w]] for w in range(32)])
print("k-entries max per row", ek.max(0))
