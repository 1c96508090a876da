"""Field training oracle: the binary64 restatement
or_train_grad / or_adam_update / or_lr_at, checked against the SPEC's own
oracles -- central finite differences of the loss, the lr table, the
zero-gradient example -- before the GPU trainer is compared with it."""
import numpy as np
import pytest

from paper_2304_07338_b200 import FieldConfig


def _batch(n, seed=0):
    r = np.random.default_rng(seed)
    return (r.random((n, 3)), r.random((n, 2)), r.choice([-0.75, 0.0, 0.75], n), r.random((n, 3)))


@pytest.mark.parametrize("cfg", ["desk", "tiny"])
def test_gradient_matches_finite_differences(oracle, cfg):
    """analytic gradient vs central differences (binary64, 64-parameter
    random subset, h = 1e-4): max relative error < 1e-3.  The rMSE denominator is
    the detached prediction, so it is frozen for the differences."""
    if cfg == "desk":
        fc = FieldConfig.desk()
    else:
        from paper_2304_07338_b200 import HashGrid
        fc = FieldConfig(pos=HashGrid(3, 2, 4, 2, 2.0, 6), dir=HashGrid(2, 2, 4, 2, 2.0, 6), hidden_layers=2)
    p = fc.init_params(seed=3, embed_scale=0.3, bias_scale=0.1).astype(np.float64)
    x, w, g, t = _batch(64)
    loss, grad, touched, pred = oracle.train_grad(fc, p, x, w, g, t, want_pred=True)
    den = pred ** 2 + 0.01
    n_tab = len(p) - oracle._mlp_count(fc)
    r = np.random.default_rng(1)
    cand = np.concatenate([np.flatnonzero(grad[:n_tab] != 0), np.arange(n_tab, len(p))])
    idx = r.choice(cand, 64, replace=False)
    def fd(i, h):
        pp = p.copy()
        pp[i] += h
        lp = oracle.train_grad(fc, pp, x, w, g, t, want_grad=False, den=den)[0]
        pp[i] -= 2 * h
        lm = oracle.train_grad(fc, pp, x, w, g, t, want_grad=False, den=den)[0]
        return (lp - lm) / (2 * h)

    def rel(a, b):
        return abs(a - b) / max(abs(a), abs(b), 1e-8)

    worst = 0.0
    for i in idx:
        e = rel(fd(i, 1e-4), grad[i])
        if e >= 1e-3:
            # a ReLU kink inside [-h, h] (the loss is piecewise smooth in the
            # weights): the derivative is still defined at p, so re-difference
            # at a step that stays on one side of the kink
            e = rel(fd(i, 1e-7), grad[i])
        worst = max(worst, e)
    assert worst < 1e-3, worst
    # untouched table entries have exactly zero gradient
    mask = np.repeat(touched.astype(bool), fc.pos.features)
    assert touched.sum() > 0 and not np.any(grad[:n_tab][~mask])


def test_lr_schedule_table(oracle):
    """lr(step) = 9e-4 * 0.92^floor(max(0, step - 0.7 T) / 25), T = 3000."""
    got = [oracle.lr_at(s, 3000) for s in (0, 2099, 2100, 2125, 3000)]
    assert np.allclose(got, [9e-4, 9e-4, 9e-4, 8.28e-4, 4.473055573e-5], rtol=1e-9)


def test_zero_gradient_step_leaves_parameters(oracle):
    """targets equal the current predictions -> loss 0 and the Adam
    step changes no parameter by more than epsilon effects (< 1e-6)."""
    fc = FieldConfig.desk()
    p = fc.init_params(seed=5, embed_scale=0.2, bias_scale=0.1).astype(np.float64)
    x, w, g, _ = _batch(128, 2)
    _, _, _, pred = oracle.train_grad(fc, p, x, w, g, np.zeros((128, 3)), want_pred=True)
    loss, grad, touched = oracle.train_grad(fc, p, x, w, g, pred)
    assert loss == 0.0 and not grad.any()
    q = p.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam_update(fc, q, grad, touched, m, v, 0, 100)
    assert np.max(np.abs(q - p)) < 1e-6


def test_sparse_adam_only_touches_visited_entries(oracle):
    fc = FieldConfig.desk()
    p = fc.init_params(seed=6, embed_scale=0.2, bias_scale=0.1).astype(np.float64)
    x, w, g, t = _batch(16, 3)
    loss, grad, touched = oracle.train_grad(fc, p, x, w, g, t)
    q = p.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam_update(fc, q, grad, touched, m, v, 0, 100)
    n_tab = len(p) - oracle._mlp_count(fc)
    changed = q[:n_tab] != p[:n_tab]
    # entries -> parameter mask (desk: 4 features for both grids)
    mask = np.repeat(touched.astype(bool), fc.pos.features)
    assert not np.any(changed & ~mask)
    assert np.all(q[n_tab:] != p[n_tab:]) or np.count_nonzero(grad[n_tab:] == 0) > 0
    assert loss > 0


def test_checkpoint_file_roundtrip(tmp_path):
    from paper_2304_07338_b200 import AdamConfig, checkpoint_training_state, load_checkpoint, lr_at, save_checkpoint
    fc = FieldConfig.desk()
    p = fc.init_params(seed=2, embed_scale=0.2)
    m, v = p * 0.5, np.abs(p) * 1e-3
    f = tmp_path / "x.pffc"
    adam = AdamConfig(lr=1e-3, beta2=0.999, decay_interval=7, eps_rel=0.02)
    save_checkpoint(f, fc, [-0.75, 0.0, 0.75], 12, p, m, v, adam=adam, total_steps=40)
    cfg, gs, step, p2, m2, v2 = load_checkpoint(f)
    assert cfg == fc and gs == [-0.75, 0.0, 0.75] and step == 12
    assert checkpoint_training_state(f) == (adam, 40)
    for a, b in ((p, p2), (m, m2), (v, v2)):
        assert np.array_equal(a.astype(np.float64), b)
    f.write_bytes(f.read_bytes()[:-8])
    with pytest.raises(ValueError):
        load_checkpoint(f)
    assert [lr_at(s, 3000) for s in (0, 2125, 3000)] == pytest.approx([9e-4, 8.28e-4, 4.473055573e-5], rel=1e-9)


def test_checkpoint_version1_still_loads(tmp_path):
    """Round-1 checkpoints (version 1: no Adam block) load; their Adam config
    and total_steps read as unknown (None, 0)."""
    import struct
    from paper_2304_07338_b200 import checkpoint_training_state, load_checkpoint
    fc = FieldConfig.desk()
    p = fc.init_params(seed=4, embed_scale=0.1)
    m, v = p * 0.25, np.abs(p) * 1e-4
    gs = np.array([-0.75, 0.0, 0.75])
    f = tmp_path / "v1.pffc"
    with open(f, "wb") as fh:  # the version-1 layout, written by hand
        fh.write(b"PFFC" + struct.pack("<I", 1))
        for hg in (fc.pos, fc.dir):
            fh.write(struct.pack("<iiiidi", hg.dims, hg.levels, hg.features, hg.base_res, float(hg.growth),
                                 hg.log2_table))
        fh.write(struct.pack("<iid", fc.hidden_layers, fc.width, float(fc.psi)))
        fh.write(struct.pack("<I", len(gs)) + gs.astype("<f8").tobytes())
        fh.write(struct.pack("<QQ", 7, len(p)))
        for arr in (p, m, v):
            fh.write(np.asarray(arr, np.float64).astype("<f8").tobytes())
    cfg, g2, step, p2, m2, v2 = load_checkpoint(f)
    assert cfg == fc and g2 == list(gs) and step == 7
    assert np.array_equal(p2, p.astype(np.float64)) and np.array_equal(v2, v.astype(np.float64))
    assert checkpoint_training_state(f) == (None, 0)
