"""GPU: the pipelined sequence step (recycle.solve_next_async + job.finish,
used by the def-CG Newton loop) against the synchronous solve_next, which is
itself checked against the reference (test_gpu_recycle.py).

The pipelined path moves three host decisions onto the device: the refresh's
surviving column count (the solve kernel reads it), the extraction's sizes
(read from the solve's status block) and BasisDeficient (a column count of 0,
i.e. plain CG, recycle.py:178-179, 194-195).  These tests pin each of them to
the synchronous semantics on identical inputs."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1706_00241_b200 as P

    return P


def gpc_like_sequence(P, n, steps, seed=0):
    """A = I + S_t K S_t with K an RBF Gram and slowly varying s_t (the
    Laplace-Newton system shape), b_t random."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 5))
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.5))
    s0 = rng.uniform(0.2, 0.5, n)
    systems = []
    for t in range(steps):
        s = torch.from_numpy(s0 * (1.0 + 0.05 * t * rng.uniform(-1, 1, n))).cuda()
        b = torch.from_numpy(rng.standard_normal(n)).cuda()
        systems.append((gram.scaled(s, 1.0), b))
    return systems


def run_sync(P, systems, k, cfg):
    st = P.SequenceState(k=k, cfg=cfg, selection="largest")
    xs, its = [], []
    for a, b in systems:
        x, st = P.solve_next(st, a, b)
        xs.append(x.clone())
        its.append(st.history[-1].iterations)
    return xs, its


def run_pipelined(P, systems, k, cfg):
    st = P.SequenceState(k=k, cfg=cfg, selection="largest")
    xs, its = [], []
    for a, b in systems:
        _, job = P.recycle.solve_next_async(st, a, b)
        x, st = job.finish()
        xs.append(x.clone())
        its.append(st.history[-1].iterations)
    _ = st.basis
    return xs, its


@pytest.mark.parametrize("n,k,ell", [(800, 8, 12), (1500, 16, 20)])
def test_pipelined_sequence_matches_sync(P, n, k, ell):
    systems = gpc_like_sequence(P, n, 6)
    cfg = P.SolverConfig(tol=1e-8, ell=ell)
    xs_s, its_s = run_sync(P, systems, k, cfg)
    xs_p, its_p = run_pipelined(P, systems, k, cfg)
    assert all(abs(a - b) <= 1 for a, b in zip(its_s, its_p)), (its_s, its_p)
    for a, b in zip(xs_s, xs_p):
        assert float(torch.linalg.norm(a - b) / torch.linalg.norm(a)) <= 1e-9
    # recycling engaged after the first system (fewer iterations than plain CG)
    assert its_p[-1] < its_p[0]


def test_pipelined_first_solve_is_plain_cg_bitwise(P):
    """No basis yet: the pipelined first solve is exactly cg_solve (k = 0 path)."""
    systems = gpc_like_sequence(P, 600, 1)
    cfg = P.SolverConfig(tol=1e-8, ell=10)
    a, b = systems[0]
    x_ref, rep_ref, _ = P.cg_solve(a, b, torch.zeros_like(b), cfg)
    st = P.SequenceState(k=6, cfg=cfg, selection="largest")
    _, job = P.recycle.solve_next_async(st, a, b)
    x, st = job.finish()
    assert torch.equal(x, x_ref)
    assert st.history[-1].residual_history == rep_ref.residual_history


def test_failed_extraction_means_plain_cg(P):
    """An extraction that reports BasisDeficient (device result block) makes
    the pipelined refresh leave 0 columns: the next solve is plain CG from
    the previous solution, exactly as solve_next after a swallowed
    BasisDeficient (recycle.py:194-195)."""
    systems = gpc_like_sequence(P, 700, 2)
    cfg = P.SolverConfig(tol=1e-8, ell=12)
    st = P.SequenceState(k=8, cfg=cfg, selection="largest")
    _, job = P.recycle.solve_next_async(st, *systems[0])
    x0, st = job.finish()
    pending = object.__getattribute__(st, "basis")
    pending.join(torch.cuda.current_stream())
    pending.event.synchronize()
    pending.result[0] = P._native.DCG_E_BASIS_DEFICIENT   # as the device would have written it
    _, job = P.recycle.solve_next_async(st, *systems[1])
    x1, st1 = job.finish()
    assert job.log.k == 0
    x_ref, rep_ref, _ = P.cg_solve(systems[1][0], systems[1][1], x0, cfg)
    assert torch.equal(x1, x_ref)
    assert st1.history[-1].iterations == rep_ref.iterations


def test_deficient_extraction_on_device(P):
    """k > k_prev + m (a solve that stops after fewer than k iterations with no
    previous basis): the device-side check yields BasisDeficient, the next
    solve runs plain CG -- the same outcome the synchronous path reaches."""
    n = 400
    rng = np.random.default_rng(3)
    d = np.linspace(1.0, 2.0, n)
    a = torch.diag(torch.from_numpy(d)).cuda()
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    cfg = P.SolverConfig(tol=1e-3, ell=20)
    st = P.SequenceState(k=16, cfg=cfg, selection="largest")
    _, job = P.recycle.solve_next_async(st, a, b)
    _, st = job.finish()
    its = st.history[-1].iterations
    assert its < 16
    assert st.basis is None   # resolves the device result: BasisDeficient, swallowed
    ss = P.SequenceState(k=16, cfg=cfg, selection="largest")
    _, ss = P.solve_next(ss, a, b)
    assert ss.basis is None


@pytest.mark.parametrize("strategy", ["sym", "sym_rowmajor", "rows"])
@pytest.mark.parametrize("n", [300, 1000, 2113, 4500])
def test_fused_newton_system_matches_separate_products(P, n, strategy):
    """dcg_gpc_newton_system_ax0 (b and ax0 = A x_prev from one pass over a
    symmetric-stored K, sym_pass1<NV = 2>) equals newton_system followed by
    the operator's own A x_prev bitwise: same tile partition, same partial
    layout, same pass-2 order."""
    from paper_1706_00241_b200 import gpc as G

    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 4))
    gram = P.rbf_kernel(torch.from_numpy(x).cuda(), P.KernelParams(1.0, 1.3)).with_strategy(strategy)   # "sym": the fused pass
    y = np.where(rng.standard_normal(n) > 0, 1.0, -1.0)
    state = G.make_state(gram, torch.from_numpy(y).cuda())
    state.f = torch.from_numpy(rng.standard_normal(n)).cuda()
    state.grad_loglik = torch.from_numpy(rng.standard_normal(n)).cuda()
    state.h = torch.from_numpy(rng.uniform(0.05, 0.25, n)).cuda()
    x_prev = torch.from_numpy(rng.standard_normal(n)).cuda()
    fused = G.build_newton_system(state, x_prev=x_prev)
    plain = G.build_newton_system(state)
    ax0 = plain.a_matrix.matvec_dev(x_prev)
    torch.cuda.synchronize()
    assert torch.equal(fused.sqrt_h, plain.sqrt_h) and torch.equal(fused.inner, plain.inner)
    assert torch.equal(fused.b, plain.b)
    assert torch.equal(fused.ax0, ax0)
    # and against fp64 torch on the dense Gram
    kd = gram.dense_dev()[:n, :n]
    s = plain.sqrt_h
    assert torch.allclose(fused.ax0, x_prev + s * (kd @ (s * x_prev)), rtol=1e-12, atol=1e-11)
    assert torch.allclose(fused.b, s * (kd @ plain.inner), rtol=1e-12, atol=1e-11)


def test_interleaved_pipelined_sequences(P):
    """Two pipelined sequences advanced alternately (each one's extraction
    tail still pending when the other enqueues its own into the shared slot-1
    workspace): every solve equals the same sequence run alone, bitwise."""
    sa = gpc_like_sequence(P, 900, 5, seed=1)
    sb = gpc_like_sequence(P, 700, 5, seed=2)
    cfg = P.SolverConfig(tol=1e-8, ell=12)
    xa_ref, ita_ref = run_pipelined(P, sa, 8, cfg)
    xb_ref, itb_ref = run_pipelined(P, sb, 8, cfg)
    st_a = P.SequenceState(k=8, cfg=cfg, selection="largest")
    st_b = P.SequenceState(k=8, cfg=cfg, selection="largest")
    xa, xb, ita, itb = [], [], [], []
    for (a1, b1), (a2, b2) in zip(sa, sb):
        _, ja = P.recycle.solve_next_async(st_a, a1, b1)
        _, jb = P.recycle.solve_next_async(st_b, a2, b2)   # enqueued before A's job finishes
        x1, st_a = ja.finish()
        x2, st_b = jb.finish()
        xa.append(x1.clone())
        xb.append(x2.clone())
        ita.append(st_a.history[-1].iterations)
        itb.append(st_b.history[-1].iterations)
    _ = st_a.basis, st_b.basis
    assert ita == ita_ref and itb == itb_ref
    for u, v in zip(xa + xb, xa_ref + xb_ref):
        assert torch.equal(u, v)
