"""Generator checks (CPU): determinism, row independence, realized sparsity vs target, grid bounds."""
import numpy as np
import pytest

import oracle
import synth


def test_deterministic_and_row_independent():
    cfg = synth.CONFIGS["1B"].replace(M=64, K=256, N=512, Kb=16)
    a = synth.gen_x(cfg)
    b = synth.gen_x(cfg)
    assert np.array_equal(a, b)
    rows = [0, 5, 63]
    assert np.array_equal(synth.gen_x_rows(cfg, rows), a[rows])
    w = synth.gen_w(cfg, "g")
    assert np.array_equal(synth.gen_w(cfg, "g", 100, 10), w[100:110])
    assert not np.array_equal(synth.gen_x(cfg.replace(seed=1)), a)


def test_grid_bounds():
    cfg = synth.CONFIGS["1B"].replace(M=32, N=256)
    qx = np.rint(synth.bf16_to_f32(synth.gen_x(cfg)) * 2 ** cfg.x_exp)
    assert np.abs(qx).max() <= 14
    for w in "gud":
        qw = np.rint(synth.bf16_to_f32(synth.gen_w(cfg, w)) * 2 ** cfg.w_exp)
        assert np.abs(qw).max() <= 7


@pytest.mark.parametrize("name,rows", [("tiny", None), ("1B", 256), ("7B", 96)])
def test_realized_sparsity(name, rows):
    """Mean density of relu(X W_g^T) within 5% relative of the target on a row sample spread over the batch."""
    cfg = synth.CONFIGS[name]
    p = synth.token_targets(cfg)
    if rows is None:
        idx = np.arange(cfg.M)
    else:
        idx = np.random.default_rng(0).choice(cfg.M, rows, replace=False)
    X = synth.gen_x_rows(cfg, idx, p=p)
    Wg = synth.gen_w(cfg, "g")
    A = oracle.gate_preact(X, Wg)
    dens = (A > 0).mean(1)
    target = p[idx].mean()
    assert abs(dens.mean() - target) / target < 0.05 + 2.0 / np.sqrt(len(idx) * cfg.N * target)
    # heavy tail: the densest sampled token is well above the mean
    if cfg.tok_sigma > 0 and rows:
        assert dens.max() > 2.0 * dens.mean()


def test_dead_neurons():
    cfg = synth.CONFIGS["1B"].replace(M=128, K=512, N=1024, Kb=16)
    b, dead = synth.neuron_params(cfg)
    assert abs(dead.mean() - cfg.dead_frac) < 0.05
    A = oracle.gate_preact(synth.gen_x(cfg), synth.gen_w(cfg, "g"))
    assert not np.any(A[:, dead.astype(bool)] > 0)


def test_neuron_popularity_lognormal():
    """per-neuron popularity (the fraction of tokens a live neuron fires for) is lognormal with
    sigma ~ 1 (std of log popularity over the live neurons of a 2048-token window of the 7B config), with hot
    neurons (small beta) firing far more often than cold ones."""
    cfg = synth.CONFIGS["7B"]
    p = synth.token_targets(cfg)
    A = oracle.gate_preact_matmul(synth.gen_x(cfg, 0, 2048, p=p), synth.gen_w(cfg, "g"))
    pop = (A > 0).mean(0)
    bq, dead = synth.neuron_params(cfg)
    alive = pop > 0
    assert abs(alive.mean() - (1 - cfg.dead_frac)) < 0.05 and not np.any(pop[dead.astype(bool)] > 0)
    s = np.std(np.log(pop[alive]))
    assert 0.8 < s < 1.25, s
    live = ~dead.astype(bool)
    hot, cold = bq[live] <= np.percentile(bq[live], 10), bq[live] >= np.percentile(bq[live], 90)
    assert pop[live][hot].mean() > 10 * pop[live][cold].mean()


def test_direct_pattern_mode():
    """Direct mode: per-token density follows the targets, popularity follows the lognormal weights, values are
    positive grid values; deterministic and row-independent."""
    cfg = synth.CONFIGS["7B"].replace(M=4096)
    p = synth.token_targets(cfg)
    H = synth.gen_pattern(cfg, p=p)
    assert np.array_equal(synth.gen_pattern(cfg, 100, 7, p=p), H[100:107])
    act = H != 0
    assert abs(act.mean() - p.mean()) / p.mean() < 0.03
    assert np.corrcoef(act.mean(1), p)[0, 1] > 0.9
    v = synth.bf16_to_f32(H[act]) * 16
    assert (v >= 1).all() and (v <= 15).all() and np.array_equal(v, np.rint(v))
    pop = act.mean(0)
    assert np.std(np.log(pop[pop > 0])) > 0.7
