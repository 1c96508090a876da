"""Field training on the GPU vs the binary64 oracle.

Tolerances: the trainer keeps binary32 master parameters / activations and
accumulates table gradients in 2^-40 fixed point, the oracle is binary64
throughout, so
  * loss: relative 1e-5;
  * gradient: |g_gpu - g_oracle| <= 2e-3 |g_oracle| + 1e-5 max|g_oracle| per
    component; touched-entry flags identical;
  * one Adam step: the update of every component whose gradient is well
    above binary32 noise (|g| > 1e-3 max|g|) within 1e-3 relative; untouched
    table entries bit-unchanged;
  * determinism: repeated steps are bit-identical (fixed reduction order).
"""
import numpy as np
import pytest

from paper_2304_07338_b200 import AdamConfig, FieldConfig, TrainConfig
from paper_2304_07338_b200.scene import default_lights, synth_volume, tf_scene_b

pytestmark = pytest.mark.gpu


def _batch(n, seed=0):
    r = np.random.default_rng(seed)
    x = r.random((n, 3)).astype(np.float32)
    w = r.random((n, 2)).astype(np.float32)
    g = r.choice([-0.75, 0.0, 0.75], n).astype(np.float32)
    t = r.random((n, 3)).astype(np.float32)
    return x, w, g, t


@pytest.mark.parametrize("cfg", ["desk", "paper"])
def test_gradient_matches_oracle(ctx, oracle, cfg):
    fc = FieldConfig.desk() if cfg == "desk" else FieldConfig.paper()
    params = fc.init_params(seed=7, embed_scale=0.1, bias_scale=0.05)
    ctx.train_init(fc, params)
    n = 2048 if cfg == "desk" else 512
    x, w, g, t = _batch(n, 1)
    loss, grad, touched = ctx.train_grad(x, w, g, t)
    oloss, ograd, otouched = oracle.train_grad(fc, params.astype(np.float64), x.astype(np.float64),
                                               w.astype(np.float64), g.astype(np.float64), t.astype(np.float64))
    print(cfg, "loss", loss, oloss)
    assert abs(loss - oloss) <= 1e-5 * oloss
    assert np.array_equal(touched, otouched)
    scale = np.abs(ograd).max()
    bad = np.abs(grad - ograd) > 2e-3 * np.abs(ograd) + 1e-5 * scale
    print("grad mismatches", np.count_nonzero(bad), "of", len(grad), "max|g|", scale)
    assert not np.any(bad)
    # bit-reproducible
    loss2, grad2, _ = ctx.train_grad(x, w, g, t)
    assert loss2 == loss and np.array_equal(grad2.view(np.uint32), grad.view(np.uint32))


def test_adam_step_matches_oracle(ctx, oracle):
    fc = FieldConfig.desk()
    params = fc.init_params(seed=8, embed_scale=0.1, bias_scale=0.05)
    ctx.train_init(fc, params)
    x, w, g, t = _batch(1024, 2)
    loss = ctx.train_step(x, w, g, t, step=0, total_steps=100)
    new = ctx.train_params()
    p64 = params.astype(np.float64)
    oloss, ograd, otouched = oracle.train_grad(fc, p64, x.astype(np.float64), w.astype(np.float64),
                                               g.astype(np.float64), t.astype(np.float64))
    q = p64.copy()
    m, v = np.zeros_like(q), np.zeros_like(q)
    oracle.adam_update(fc, q, ograd, otouched, m, v, 0, 100)
    assert abs(loss - oloss) <= 1e-5 * oloss
    n_tab = len(q) - oracle._mlp_count(fc)
    mask = np.repeat(otouched.astype(bool), fc.pos.features)
    assert np.array_equal(new[:n_tab][~mask].view(np.uint32), params[:n_tab][~mask].view(np.uint32))
    sig = np.abs(ograd) > 1e-3 * np.abs(ograd).max()
    du, dq = new.astype(np.float64) - params, q - p64
    err = np.abs(du[sig] - dq[sig]) / np.abs(dq[sig])
    print("adam: compared", sig.sum(), "max rel err", err.max())
    assert err.max() < 1e-3


def test_training_is_deterministic(ctx):
    fc = FieldConfig.desk()
    params = fc.init_params(seed=9, embed_scale=0.1, bias_scale=0.05)
    runs = []
    for _ in range(2):
        ctx.train_init(fc, params)
        for s in range(5):
            ctx.train_step(*_batch(4096, 10 + s), step=s, total_steps=5)
        runs.append(ctx.train_params())
    assert np.array_equal(runs[0].view(np.uint32), runs[1].view(np.uint32))


def test_overfit_fixed_batch(ctx):
    """fixed 1024-sample batch, 2000 steps -> loss < 1e-3."""
    fc = FieldConfig.desk()
    ctx.train_init(fc, fc.init_params(seed=1, embed_scale=1e-4, bias_scale=0.0))
    x, w, g, t = _batch(1024, 5)
    losses = [ctx.train_step(x, w, g, t, step=s, total_steps=2000) for s in range(2000)]
    print("overfit loss", losses[0], losses[100], losses[-1])
    assert losses[-1] < 1e-3


def test_train_argument_errors(ctx):
    fc = FieldConfig.desk()
    with pytest.raises(ValueError, match="AdamState"):
        ctx.train_init(fc, fc.init_params(seed=1), AdamConfig(lr=-1.0))
    ctx.train_init(fc, fc.init_params(seed=1))
    with pytest.raises(ValueError, match="step"):
        ctx.train_step(*_batch(8), step=5, total_steps=5)
    with pytest.raises(ValueError, match="KnnSchedule"):
        ctx.train(TrainConfig(total_steps=2, batch_size=16, K=8, schedule_ends=(0.5, 0.9)))


@pytest.fixture(scope="module")
def traced_map(ctx):
    """A photon map traced on the device through the config-1 style scene."""
    from paper_2304_07338_b200 import TraceConfig
    ctx.upload_volume(synth_volume("sphere_sinusoid", 64))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    tc = TraceConfig(n_total=400_000, seed=2)
    ctx.trace_photons(tc, device=True)
    ctx.knn_build_traced(tc.phase_set)
    return tc


def test_train_loop_on_traced_map(ctx, traced_map):
    """the staggered loop learns (late loss < early loss), the
    KNN sampling time is reported, the trained field renders."""
    from paper_2304_07338_b200 import RenderConfig
    from paper_2304_07338_b200.scene import CameraSpec
    fc = FieldConfig.desk()
    ctx.train_init(fc, fc.init_params(seed=3, embed_scale=1e-4, bias_scale=0.0))
    cfg = TrainConfig(total_steps=400, batch_size=4096, K=64, schedule_ends=(0.36, 0.63, 0.9, 1.0),
                      schedule_radii=(0.05, 0.1, 0.2, 0.4), seed=4)
    res = ctx.train(cfg)
    h = res.loss_history
    print("loss", h[:3], h[-3:], "knn ms", res.knn_ms, "step ms", res.step_ms)
    assert np.all(np.isfinite(h))
    assert np.median(h[-20:]) < 0.5 * np.median(h[5:25])
    assert res.knn_ms > 0 and res.step_ms > 0
    img = ctx.render_neural(CameraSpec(64, 48), RenderConfig(spp=2, g=0.0, seed=1, mode="fast"))
    assert np.all(np.isfinite(img)) and img.mean() > 0


def test_staggered_schedule_is_cheaper(ctx, traced_map):
    """staggered vs naive (single segment at the final radius): final
    losses within 15%, staggered cumulative KNN time strictly lower."""
    fc = FieldConfig.desk()
    out = {}
    for name, ends, radii in [("staggered", (0.36, 0.63, 0.9, 1.0), (0.05, 0.1, 0.2, 0.4)),
                              ("naive", (1.0,), (0.4,))]:
        ctx.train_init(fc, fc.init_params(seed=3, embed_scale=1e-4, bias_scale=0.0))
        out[name] = ctx.train(TrainConfig(total_steps=300, batch_size=4096, K=256, schedule_ends=ends,
                                          schedule_radii=radii, seed=4))
    s, n = out["staggered"], out["naive"]
    ls, ln = np.median(s.loss_history[-20:]), np.median(n.loss_history[-20:])
    print("final loss", ls, ln, "knn ms", s.knn_ms, n.knn_ms)
    assert s.knn_ms < n.knn_ms
    assert abs(ls - ln) <= 0.15 * max(ls, ln) or ls < ln


def test_checkpoint_resume_is_bit_exact(ctx, tmp_path):
    """a field checkpoint (params + Adam moments, binary64 on disk)
    restores training bit-exactly."""
    fc = FieldConfig.desk()
    ctx.train_init(fc, fc.init_params(seed=11, embed_scale=0.1, bias_scale=0.05))
    batches = [_batch(2048, 40 + s) for s in range(6)]
    for s in range(3):
        ctx.train_step(*batches[s], step=s, total_steps=6)
    ckpt = tmp_path / "field.pffc"
    ctx.train_save(ckpt, [-0.75, 0.0, 0.75], 3)
    for s in range(3, 6):
        ctx.train_step(*batches[s], step=s, total_steps=6)
    a = ctx.train_state()
    cfg, gs, nxt = ctx.train_load(ckpt)
    assert cfg == fc and nxt == 3 and gs == [-0.75, 0.0, 0.75]
    for s in range(nxt, 6):
        ctx.train_step(*batches[s], step=s, total_steps=6)
    b = ctx.train_state()
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_training_log(ctx, traced_map, tmp_path):
    """one line per step -- step, loss, radius, lr, cumulative knn_time."""
    fc = FieldConfig.desk()
    ctx.train_init(fc, fc.init_params(seed=3, embed_scale=1e-4, bias_scale=0.0))
    res = ctx.train(TrainConfig(total_steps=40, batch_size=1024, K=32, schedule_ends=(0.5, 1.0),
                                schedule_radii=(0.1, 0.2), seed=1))
    log = tmp_path / "train.csv"
    res.write_log(log)
    rows = log.read_text().strip().splitlines()
    assert rows[0] == "step,loss,radius,lr,knn_time_ms" and len(rows) == 41
    cols = np.array([[float(v) for v in r.split(",")] for r in rows[1:]])
    assert np.array_equal(cols[:, 0], np.arange(40))
    assert set(cols[:, 2]) == {0.1, 0.2} and np.all(np.diff(cols[:, 4]) >= 0)
    assert abs(res.knn_ms - res.knn_ms_steps.sum()) < 1e-6 * max(1.0, res.knn_ms)


def test_train_resume_through_checkpoint(ctx, traced_map, tmp_path):
    """SPEC.md:439 through the public loop: train(stop=k) -> train_save ->
    train_load (Adam hyperparameters from the checkpoint) -> train(start=k) is
    bit-identical to one uninterrupted train() -- same parameters, moments
    and per-step losses (the radius schedule, query streams, lr and bias
    correction all continue at the absolute step)."""
    from paper_2304_07338_b200 import checkpoint_training_state
    fc = FieldConfig.desk()
    adam = AdamConfig(lr=2e-3, decay_start=0.5, decay_interval=3)
    tc = TrainConfig(total_steps=12, batch_size=1024, K=32, schedule_ends=(0.5, 1.0), schedule_radii=(0.1, 0.2),
                     seed=5)
    p0 = fc.init_params(seed=3, embed_scale=1e-2, bias_scale=0.0)
    ctx.train_init(fc, p0, adam)
    full = ctx.train(tc)
    a = ctx.train_state()
    ctx.train_init(fc, p0, adam)
    first = ctx.train(tc, stop_step=5)
    assert first.first_step == 0 and len(first.loss_history) == 5
    ck = tmp_path / "chunk.pffc"
    ctx.train_save(ck, ctx.phase_set, 5, tc.total_steps)
    assert checkpoint_training_state(ck) == (adam, 12)
    ctx.train_init(fc, fc.init_params(seed=99, embed_scale=0.5))  # clobber the optimizer state
    cfg, gs, nxt = ctx.train_load(ck)
    assert cfg == fc and nxt == 5 and ctx.adam_config == adam
    rest = ctx.train(tc, start_step=nxt)
    assert rest.first_step == 5 and len(rest.loss_history) == 7
    b = ctx.train_state()
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert np.array_equal(np.concatenate([first.loss_history, rest.loss_history]), full.loss_history)
    log = tmp_path / "rest.csv"
    rest.write_log(log)
    assert log.read_text().splitlines()[1].startswith("5,")
