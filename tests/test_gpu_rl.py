"""GPU parity of NEXT-2, the actor-critic scheduler (reading S3): environment
transitions bit-exact against oracle.env_rollout (forced and sampled actions), the policy's sampling
distribution, the actor-critic gradient against the oracle's fp64 gradient, and a short training run."""
import numpy as np
import pytest

import oracle
from bench import lat_profile
from test_oracle_rl import gold

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TAU = 560_000_000


@pytest.fixture(scope="module")
def rk():
    import paper_1804_06087_b200 as m
    m.load_library()
    return m


def make(rk, K, B, ref=572.0, N=200_000, L=16, H=32, n=24, seed=5):
    ctx = rk.Context(0)
    ctx.load_ensemble(K, 10)
    arr = torch.empty(N, dtype=torch.int64, device="cuda")
    ctx.sine_arrivals(arr, N, ref, 500 * TAU, 50_000_000, 0.1, seed)
    cfg = rk.RewardCfg(B=B, beta=1.0, tau_ns=TAU, lat_ns=lat_profile(K, B), rates=[1.0])
    acc = np.sort(np.random.default_rng(K).uniform(0.7, 0.9, (1 << K) - 1))
    ac = {"L": L, "H": H, "n_steps": n, "gamma": 0.9, "reward_scale": 1.0 / max(B)}
    return ctx, arr, cfg, acc, ac


def traj(E, n, F):
    return {"states": torch.zeros((E, n, F), dtype=torch.float32, device="cuda"),
            "actions": torch.zeros((E, n), dtype=torch.int32, device="cuda"),
            "rewards": torch.zeros((E, n), dtype=torch.float64, device="cuda"),
            "overdue": torch.zeros((E, n), dtype=torch.int32, device="cuda"),
            "t_dec": torch.zeros((E, n), dtype=torch.int64, device="cuda"),
            "t_start": torch.zeros((E, n), dtype=torch.int64, device="cuda"),
            "t_done": torch.zeros((E, n), dtype=torch.int64, device="cuda")}


def check_against_oracle(tr, K, cfg, acc, arr_np, L, h0):
    E, n = tr["actions"].shape
    for e in range(E):
        o = oracle.env_rollout(K, cfg.B, cfg.lat_ns, TAU, 1.0, acc, arr_np, L, tr["actions"][e].cpu().numpy(),
                               int(h0[e]))
        np.testing.assert_array_equal(tr["rewards"][e].cpu().numpy(), o["rewards"])
        np.testing.assert_array_equal(tr["states"][e].cpu().numpy(), o["states"])
        for k in ("overdue", "t_dec", "t_start", "t_done"):
            np.testing.assert_array_equal(tr[k][e].cpu().numpy(), o[k], err_msg=k)


def test_hand_worked(rk):
    g = gold()
    ctx = rk.Context(0)
    ctx.load_ensemble(2, 10)
    arr = torch.tensor(np.array(g["arrivals"], np.int64)).cuda()
    cfg = rk.RewardCfg(B=[1, 2], beta=1.0, tau_ns=50, lat_ns=np.array([[10, 15], [30, 40]]), rates=[1.0])
    ac = {"L": 2, "H": 4, "n_steps": 3, "gamma": 0.9, "reward_scale": 1.0}
    F, A, P = ctx.ac_dims(2, ac)
    assert (F, A) == (8, 6)
    tr = traj(1, 3, F)
    forced = torch.tensor([[int(a) for a in g["actions"]]], dtype=torch.int32).cuda()
    ctx.ac_rollout(cfg, [0.9, 0.6, 0.95], arr, arr.numel(), ac, torch.zeros(P, device="cuda"), 1,
                   torch.zeros(1, dtype=torch.int64).cuda(), tr, forced=forced)
    np.testing.assert_allclose(tr["rewards"][0].cpu().numpy(), g["rewards"], rtol=0, atol=1e-12)
    for k in ("overdue", "t_dec", "t_start", "t_done"):
        assert tr[k][0].cpu().tolist() == [int(x) for x in g[k]], k
    for i in range(3):
        np.testing.assert_array_equal(tr["states"][0, i].cpu().numpy(), np.array(g[f"s{i}"], np.float32))


@pytest.mark.parametrize("K,B", [(3, [16, 32, 48, 64]), (5, [16, 32, 64, 128, 256])])
def test_forced_and_sampled_parity(rk, K, B):
    ctx, arr, cfg, acc, ac = make(rk, K, B)
    F, A, P = ctx.ac_dims(len(B), ac)
    E, n = 48, ac["n_steps"]
    rng = np.random.default_rng(K)
    h0 = torch.from_numpy(rng.integers(0, 150_000, E).astype(np.int64)).cuda()
    arr_np = arr.cpu().numpy()
    forced = torch.from_numpy(rng.integers(0, A, (E, n)).astype(np.int32)).cuda()
    tr = traj(E, n, F)
    ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, torch.zeros(P, device="cuda"), E, h0, tr, forced=forced)
    assert (tr["actions"] == forced).all()
    check_against_oracle(tr, K, cfg, acc, arr_np, ac["L"], h0.cpu().numpy())
    # sampled actions from a random policy: the same environment replays them exactly
    params = torch.from_numpy(np.random.default_rng(1).normal(0, 0.3, P).astype(np.float32)).cuda()
    tr2 = traj(E, n, F)
    ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, params, E, h0, tr2, seed=9)
    check_against_oracle(tr2, K, cfg, acc, arr_np, ac["L"], h0.cpu().numpy())
    tr3 = traj(E, n, F)
    ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, params, E, h0, tr3, seed=9)
    assert torch.equal(tr2["actions"], tr3["actions"])  # deterministic per seed


def test_uniform_policy_sampling(rk):
    """Zero parameters: pi is uniform over the (2^K - 1) * |B| actions (SPEC.md rl-agent act)."""
    K, B = 3, [16, 32, 48, 64]
    ctx, arr, cfg, acc, ac = make(rk, K, B, N=400_000, n=32)
    F, A, P = ctx.ac_dims(len(B), ac)
    E = 512
    h0 = torch.from_numpy(np.random.default_rng(0).integers(0, 300_000, E).astype(np.int64)).cuda()
    tr = traj(E, 32, F)
    ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, torch.zeros(P, device="cuda"), E, h0, tr, seed=3)
    cnt = np.bincount(tr["actions"].cpu().numpy().ravel(), minlength=A)
    m = E * 32 / A
    assert cnt.size == A and (np.abs(cnt - m) < 5 * np.sqrt(m)).all(), cnt


@pytest.mark.parametrize("K,B,H,ent", [(3, [16, 32, 48, 64], 32, 0.0), (4, [16, 64], 64, 0.0),
                                       (3, [16, 32, 48, 64], 32, 0.2)])
def test_gradient_parity(rk, K, B, H, ent):
    ctx, arr, cfg, acc, ac = make(rk, K, B, H=H, n=12)
    ac["entropy"] = ent
    F, A, P = ctx.ac_dims(len(B), ac)
    E, n = 24, 12
    params = np.random.default_rng(2).normal(0, 0.3, P).astype(np.float32)
    pd = torch.from_numpy(params).cuda()
    h0 = torch.from_numpy(np.random.default_rng(4).integers(0, 150_000, E).astype(np.int64)).cuda()
    tr = traj(E, n, F)
    ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, pd, E, h0, tr, seed=1)
    grad = torch.zeros(P, device="cuda")
    losses = ctx.ac_grad(cfg, ac, pd, tr, E, grad)
    go, lp, lv = oracle.ac_grad(F, H, A, params.astype(np.float64), tr["states"].cpu().numpy(),
                                tr["actions"].cpu().numpy(), tr["rewards"].cpu().numpy(), 0.9, 1.0 / max(B), ent)
    g = grad.cpu().numpy().astype(np.float64)
    npol = H * F + H + A * H + A
    for sl in (slice(0, npol), slice(npol, P)):  # fp32 accumulation over E*n samples vs fp64
        scale = np.abs(go[sl]).max()
        assert np.abs(g[sl] - go[sl]).max() <= 2e-4 * scale + 1e-7, (np.abs(g[sl] - go[sl]).max(), scale)
    assert abs(losses[0] - lp) <= 1e-4 * max(1.0, abs(lp)) and abs(losses[1] - lv) <= 1e-4 * max(1.0, abs(lv))
    # the SGD step moves exactly along the returned gradient
    ctx.ac_apply(cfg, ac, pd, grad, 0.5, 0.25)
    exp = params - np.concatenate([0.5 * g[:npol], 0.25 * g[npol:]]).astype(np.float32)
    np.testing.assert_allclose(pd.cpu().numpy(), exp, rtol=0, atol=1e-6)


def test_training_improves_return(rk):
    """A short actor-critic run at the paper's r_u of the trio (572 req/s): the mean episode
    return of the last iterations exceeds that of the initial (uniform) policy. Deterministic per seed."""
    from paper_1804_06087_b200.scheduler import ActorCritic
    K, B = 3, [16, 32, 48, 64]
    ctx, arr, cfg, acc, ac = make(rk, K, B, N=400_000)
    agent = ActorCritic(ctx, cfg, acc, arr, L=16, H=32, n_steps=24, seed=0)
    curve = agent.train(30, E=256, lr_pi=1.0, lr_v=0.02)
    first = curve[0]["return"]
    last = np.mean([c["return"] for c in curve[-5:]])
    assert last > first, (first, last)


def test_rollout_errors(rk):
    K, B = 3, [16, 32, 48, 64]
    ctx, arr, cfg, acc, ac = make(rk, K, B, N=20_000, n=4)
    F, A, P = ctx.ac_dims(len(B), ac)
    params = torch.zeros(P, device="cuda")
    with pytest.raises(rk.RkError):  # an episode start past the arrival array
        ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, params, 1, torch.tensor([arr.numel() + 5]).cuda(), traj(1, 4, F))
    with pytest.raises(rk.RkError):  # an episode that runs out of arrivals
        ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, params, 1, torch.tensor([arr.numel() - 20]).cuda(), traj(1, 4, F))
    with pytest.raises(rk.RkError):  # a forced action outside the action space
        ctx.ac_rollout(cfg, acc, arr, arr.numel(), ac, params, 1, torch.tensor([0]).cuda(), traj(1, 4, F),
                       forced=torch.full((1, 4), A, dtype=torch.int32).cuda())
    bad = dict(ac, H=65)
    with pytest.raises(rk.RkError):  # hidden layer wider than the kernels' register tiles
        ctx.ac_dims(len(B), bad) and ctx.ac_rollout(cfg, acc, arr, arr.numel(), bad, params, 1,
                                                    torch.tensor([0]).cuda(), traj(1, 4, F))
