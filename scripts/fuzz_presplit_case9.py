import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import phiks_oracle as O
from paper_2210_07667_b200 import PhiKS
from paper_2210_07667_b200 import workloads as W
rng = np.random.default_rng(7)
# replay the fuzz RNG up to case 9
def factor(n, k):
    if rng.integers(0, 2) == 0:
        return float(rng.uniform(0.1, 1.0)) * W.fd_dxx_neumann(n)
    return float(rng.uniform(0.1, 1.0)) * W.fd_dxx_dirichlet(n) + float(rng.uniform(-20, 20)) * W.fd_dx_dirichlet(n)
for c in range(10):
    d = int(rng.integers(2, 4))
    if d == 2:
        dims = (int(rng.choice([128, 256, 384, 512])), int(rng.choice([128, 256])))
    else:
        dims = (int(rng.choice([128, 256, 384])), int(rng.choice([128, 256])), int(rng.choice([16, 32, 48])))
    fac = [factor(n, k) for k, n in enumerate(dims)]
    mode = "same" if rng.integers(0, 2) == 0 else "lincomb"
    p = int(rng.integers(1, 5))
    ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
    nv = 1 if mode == "same" else len(ells)
    vs = [W.uniform_tensor(dims, -1.0, 1.0, seed=7000 + 11 * c + k) for k in range(nv)]
    tau = float(10 ** rng.uniform(-4, -1.5))
    ns = int(rng.integers(1, 5))
print(dims, mode, ells, tau, ns)
ref = O.phiks(fac, tau, mode, ells, vs, n_scales=ns)
refs = [W.as_flat(ref.out[(ell, j)]) for j in range(ns) for ell in ells]
for path, chain in (("i8", 1), ("i8", 0), ("dmma", 1)):
    op = PhiKS(fac); op.set_gemm_path(path); op.set_option("chain", chain)
    outs = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs], mode=mode, n_scales=ns)
    torch.cuda.synchronize()
    errs = [float(np.linalg.norm(o.cpu().numpy() - r) / np.linalg.norm(r)) for o, r in zip(outs, refs)]
    print(path, chain, ["%.2e" % e for e in errs], op.stats()["s"], op.stats()["q"])
# oracle vs dense? tiny check of oracle's own truncation: compare oracle with plan s+1
ref2 = O.phiks(fac, tau, mode, ells, vs, n_scales=ns, plan=O.Plan(ref.plan.s + 1, ref.plan.q + 2, 0))
print("oracle(s+1,q+2) vs oracle:", ["%.2e" % (np.linalg.norm(W.as_flat(ref2.out[(ell, j)]) - W.as_flat(ref.out[(ell, j)])) / np.linalg.norm(W.as_flat(ref.out[(ell, j)]))) for j in range(ns) for ell in ells])
# higher-precision check of φ_0 = e^{τK}v (x86 80-bit long double): each factor's exponential by
# Taylor scaling-and-squaring in long double, then the Tucker operator in long double
def expm_ld(X):
    X = X.astype(np.longdouble)
    nrm = np.abs(X).sum(axis=0).max()
    sig = 0 if nrm <= 0.5 else int(np.ceil(np.log2(float(nrm) / 0.5)))
    Y = X / np.longdouble(2.0) ** sig
    E = np.eye(X.shape[0], dtype=np.longdouble); term = E.copy()
    for k in range(1, 60):
        term = term @ Y / np.longdouble(k); E = E + term
    for _ in range(sig):
        E = E @ E
    return E
Ef = [expm_ld(tau * A) for A in fac]
V = vs[0].astype(np.longdouble)
T = np.einsum("ia,ab->ib", Ef[0], V.reshape(dims[0], dims[1], order="F"))
T = np.einsum("jb,ib->ij", Ef[1], T)
true0 = T.reshape(-1, order="F")
r0 = W.as_flat(ref.out[(0, 0)])
op = PhiKS(fac); op.set_gemm_path("i8")
g = op.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs], mode=mode, n_scales=ns)[0].cpu().numpy()
op2 = PhiKS(fac); op2.set_gemm_path("dmma")
g2 = op2.apply(tau, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).cuda() for v in vs], mode=mode, n_scales=ns)[0].cpu().numpy()
nt = float(np.linalg.norm(true0))
print("phi_0 vs long double: oracle %.2e  gpu i8 %.2e  gpu dmma %.2e  i8 vs dmma %.2e" % (
    float(np.linalg.norm(r0 - true0)) / nt, float(np.linalg.norm(g - true0)) / nt, float(np.linalg.norm(g2 - true0)) / nt,
    float(np.linalg.norm(g - g2)) / float(np.linalg.norm(g2))))
