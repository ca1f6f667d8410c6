"""Generate golden vectors by running the REAL reference (sparsewire 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes small ``*.npz`` fixtures next to this script.  The oracle
(``oracle/``) is checked against them by ``tests/test_oracle_golden.py`` and
the CUDA path by ``tests/test_gpu_*.py``.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from sparsewire import rng as R  # noqa: E402
from sparsewire.connectivity import (RaggedMatrix, SynVarMatrix,  # noqa: E402
                                     init_pairwise_bernoulli, remove_slots,
                                     TransposeMap, propagate_spikes)
from sparsewire.deep_r import DeepR  # noqa: E402
from sparsewire.updates import Model  # noqa: E402
from sparsewire.plasticity import Adam  # noqa: E402
from sparsewire.neurons import AlifLayer, AlifParams  # noqa: E402
from sparsewire._kernels import eprop_accumulate_batch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from golden_cases import DEEPR_CASES  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
PLANES = ("w", "grad", "adam_m", "adam_v")


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values()), "bytes")


def gen_rng():
    keys_parts = [(0,), (1,), (1, "host", 3, 7, 0), (42, "row", 0, 0, 1),
                  ("task", "example", 5), (2**64 - 1, -1, "päß-unicode-longer-than-8"),
                  (7, "init", "ff")]
    fold = np.array([R.fold_key(*p) for p in keys_parts], dtype=np.uint64)
    mix_in = np.array([0, 1, 0x9E3779B97F4A7C15, 12345, 2**63, 2**64 - 1], dtype=np.uint64)
    mix_out = np.array([R.mix64(int(x)) for x in mix_in], dtype=np.uint64)
    key = R.fold_key(9, "golden")
    rng = R.CounterRng(9, "golden")
    draws = rng.u64_array(4096)
    u01 = R.CounterRng(9, "golden").uniform01_array(4096)
    # uniform_int sequences for several n, including non powers of two
    ns = np.array([1, 2, 3, 7, 256, 700, 1000, 65536, 2**20, 3 * 2**40 + 1], dtype=np.uint64)
    ui = []
    for n in ns:
        r = R.CounterRng(9, "uint", int(n))
        ui.append([r.uniform_int(int(n)) for _ in range(512)] + [r.counter])
    ui = np.array(ui, dtype=np.uint64)
    child = np.array([R.CounterRng.from_key(key).child_key(i) for i in range(300)], dtype=np.uint64)
    # sample_k_distinct: rejection and Fisher-Yates branches
    skd_cases = [(3, 100), (10, 256), (5, 8), (8, 8), (40, 64), (1, 1), (0, 5)]
    skd = []
    for (k, n) in skd_cases:
        r = R.CounterRng(9, "skd", k, n)
        out = r.sample_k_distinct(k, n)
        skd.append(np.concatenate([out, [r.counter]]).astype(np.int64))
    save("rng.npz", fold=fold, mix_in=mix_in, mix_out=mix_out, key=np.uint64(key),
         draws=draws, u01=u01, ns=ns, ui=ui, child=child,
         skd_cases=np.array(skd_cases, dtype=np.int64),
         skd=np.array([np.pad(s, (0, 64 - s.size), constant_values=-1) for s in skd]))


def gen_remove():
    rng = np.random.default_rng(5)
    rows = []
    for _ in range(400):
        n = int(rng.integers(1, 90))
        k = int(rng.integers(0, n + 1))
        marked = np.sort(rng.choice(n, size=k, replace=False))
        m = RaggedMatrix(1, 10_000, 96)
        syn = SynVarMatrix(m, ("w",))
        m.target[0, :n] = np.arange(n) + 1000
        syn.planes["w"][0, :n] = np.arange(n) * 0.5
        m.row_length[0] = n
        remove_slots(m, syn, 0, marked)
        out = np.full(96, -1, dtype=np.int32)
        out[: m.row_length[0]] = m.target[0, : m.row_length[0]] - 1000
        mk = np.full(96, -1, dtype=np.int32)
        mk[:k] = marked
        rows.append((n, k, mk, out))
    save("remove.npz", n=np.array([r[0] for r in rows]), k=np.array([r[1] for r in rows]),
         marked=np.stack([r[2] for r in rows]), result=np.stack([r[3] for r in rows]))


def deep_r_build(num_pre, num_post, density, seed, l1, exclude_diagonal, headroom):
    """Mirrors pkg/tests/test_deep_r.py:16-37."""
    model = Model(seed)
    rng = R.CounterRng(seed, "init")

    def prob(i, cols):
        p = np.full(cols.size, density)
        if exclude_diagonal:
            p[i] = 0.0
        return p

    m, syn = init_pairwise_bernoulli(num_pre, num_post, prob, headroom, rng, var_names=PLANES)
    mask = m.slot_mask()
    w = syn.planes["w"]
    w[mask] = rng.normal_array(w.size).reshape(w.shape)[mask] * 0.1
    model.add_matrix("sg", m, syn)
    dr = DeepR(m, syn, "sg", l1_strength=l1, exclude_diagonal=exclude_diagonal)
    dr.init_bitfields(R.CounterRng(seed, "bits"))
    dr.register(model, "deep_r", "sg")
    return model, m, syn, dr


def snap(m, syn, dr):
    return dict(row_length=m.row_length.copy(), target=m.target.copy(),
                w=syn.planes["w"].copy(), grad=syn.planes["grad"].copy(),
                adam_m=syn.planes["adam_m"].copy(), adam_v=syn.planes["adam_v"].copy(),
                sign=dr.sign_bits.words.copy(), conn=dr.conn_bits.words.copy(),
                dormant=dr.dormant.copy(), last_removed=np.int64(dr.last_removed))




def gen_deep_r():
    """Per case: initial state; then per cycle: new weights (flip injection),
    l1 + group run, post state.  Mirrors test_deep_r.py:178-197."""
    for (name, P, N, dens, seed, diag, head, cycles) in DEEPR_CASES:
        model, m, syn, dr = deep_r_build(P, N, dens, seed, 0.005, diag, head)
        out = {f"init_{k}": v for k, v in snap(m, syn, dr).items()}
        out["meta"] = np.array([P, N, m.max_row_length, int(diag), cycles, seed], dtype=np.int64)
        flip = R.CounterRng(99, name)
        for c in range(cycles):
            w = syn.planes["w"]
            mask = m.slot_mask()
            scale = 0.1 if c % 2 == 0 else 1.0
            w[mask] = flip.normal_array(w.size).reshape(w.shape)[mask] * scale
            syn.planes["grad"][mask] = flip.normal_array(w.size).reshape(w.shape)[mask] * 0.01
            out[f"c{c}_w_in"] = w.copy()
            out[f"c{c}_grad_in"] = syn.planes["grad"].copy()
            dr.l1_step()
            out[f"c{c}_grad_l1"] = syn.planes["grad"].copy()
            model.run_update_group("deep_r")
            for k, v in snap(m, syn, dr).items():
                out[f"c{c}_{k}"] = v
        save(f"deepr_{name}.npz", **out)


def gen_adam():
    rng = R.CounterRng(5, "adam")
    shape = (37, 19)
    p = rng.normal_array(37 * 19).reshape(shape)
    m = np.zeros(shape)
    v = np.zeros(shape)
    out = {"p0": p.copy()}
    adam = Adam(1e-3, m=m, v=v)
    for t in range(5):
        g = rng.normal_array(37 * 19).reshape(shape) * (10.0 ** (-t))
        out[f"g{t}"] = g.copy()
        adam.apply(p, g)
        out[f"p{t + 1}"] = p.copy()
        out[f"m{t + 1}"] = m.copy()
        out[f"v{t + 1}"] = v.copy()
    save("adam.npz", **out)


def gen_alif_eprop():
    """ALIF step/surrogate (float32, neurons.py:60-73) and the numba e-prop
    kernel (_kernels.py:15-39) over several steps with ragged rows."""
    prm = AlifParams()
    rng = R.CounterRng(6, "alif")
    B, H = 8, 48
    layer = AlifLayer(H, prm, batch=B, dtype=np.float32)
    out = {}
    for t in range(6):
        rec = (rng.normal_array(B * H).reshape(B, H) * 0.4).astype(np.float32)
        ext = (rng.normal_array(B * H).reshape(B, H) * 0.4).astype(np.float32)
        out[f"rec{t}"], out[f"ext{t}"] = rec, ext
        out[f"psi{t}"] = layer.surrogate()
        layer.step(rec, ext)
        out[f"v{t}"], out[f"a{t}"], out[f"z{t}"] = layer.v.copy(), layer.a.copy(), layer.z.copy()
    # e-prop
    P, cap = 30, 12
    m = RaggedMatrix(P, H, cap)
    er = R.CounterRng(6, "eprop")
    for i in range(P):
        k = er.uniform_int(cap + 1)
        m.target[i, :k] = er.sample_k_distinct(k, H)
        m.row_length[i] = k
    eps = np.zeros((B, P, cap), dtype=np.float32)
    ebar = np.zeros_like(eps)
    grad = np.zeros((P, cap))
    a, b_, r_ = np.float32(prm.alpha), np.float32(prm.beta), np.float32(prm.rho)
    out["target"], out["row_length"] = m.target.copy(), m.row_length.copy()
    trace = np.zeros((B, P), dtype=np.float32)
    for t in range(25):
        x = (er.uniform01_array(B * P).reshape(B, P) < 0.2).astype(np.float32)
        trace *= a
        trace += x
        psi = (er.uniform01_array(B * H).reshape(B, H) * 0.5).astype(np.float32)
        lsig = er.normal_array(B * H).reshape(B, H).astype(np.float32)
        out[f"trace{t}"], out[f"psi_e{t}"], out[f"lsig{t}"] = trace.copy(), psi, lsig
        eprop_accumulate_batch(m.target, m.row_length, trace, psi, lsig, eps, ebar, grad, b_, r_, a)
    out["eps"], out["ebar"], out["grad"] = eps, ebar, grad
    save("alif_eprop.npz", **out)


def gen_transpose_prop():
    rng = R.CounterRng(8, "tp")
    P, N, cap = 50, 40, 16
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, ("g",))
    for i in range(P):
        k = rng.uniform_int(cap + 1)
        m.target[i, :k] = rng.sample_k_distinct(k, N)
        m.row_length[i] = k
        syn.planes["g"][i, :k] = rng.uniform01_array(k) * 0.2
    tm = TransposeMap(m)
    tm.rebuild()
    spikes = np.flatnonzero(rng.uniform01_array(P) < 0.3)
    out_v = np.zeros(N)
    propagate_spikes(m, syn.planes["g"], spikes, out_v)
    save("transpose_prop.npz", target=m.target, row_length=m.row_length, g=syn.planes["g"],
         col_length=tm.col_length, source_pre=tm.source_pre, source_slot=tm.source_slot,
         spikes=spikes, out=out_v)


def gen_trainer():
    """Small e-prop + DEEP R training run (classifier.py:82-263)."""
    from sparsewire.classifier import EpropClassifierTrainer, SyntheticTask
    task = SyntheticTask(num_classes=3, num_inputs=20, example_steps=60, seed=4)
    tr = EpropClassifierTrainer(task, hidden=24, batch_size=8, seed=4, deep_r=True,
                                input_density=0.3, recurrent_density=0.2)
    out = {}
    for b in range(3):
        h = tr.train_batch(b)
        out[f"b{b}_loss"] = np.float64(h["loss"])
        out[f"b{b}_acc"] = np.float64(h["accuracy"])
        out[f"b{b}_removed"] = np.int64(h["removed"])
    for name, m, syn in (("in", tr.m_in, tr.s_in), ("rec", tr.m_rec, tr.s_rec)):
        out[f"{name}_row_length"] = m.row_length.copy()
        out[f"{name}_target"] = m.target.copy()
        for pl in PLANES:
            out[f"{name}_{pl}"] = syn.planes[pl].copy()
    out["w_out"] = tr.w_out.copy()
    out["b_out"] = tr.b_out.copy()
    save("trainer.npz", **out)


def _tm_snap(model):
    out = {}
    for name in ("ff", "lat"):
        m, syn = model.net.matrices[name]
        out[f"{name}_row_length"] = m.row_length.copy()
        out[f"{name}_target"] = m.target.copy()
        out[f"{name}_g"] = syn.planes["g"].copy()
    out["updates"] = np.array([b.update_count for b in model.net.groups["rewiring"]])
    return out


def _tm_events(rule):
    kinds, dists = [], []
    for i in np.flatnonzero(rule.attempts):
        rec = rule._row_events[i]
        if rec is None:
            continue
        elim_d, form_d = rec[0], rec[1]
        kinds += [1] * len(elim_d) + [2] * len(form_d)
        dists += list(elim_d) + list(form_d)
    return np.array(kinds, dtype=np.int8), np.array(dists, dtype=np.float64)


def gen_topomap():
    """State-injection fixtures for the rewiring rule: the full ff/lat state
    before and after each rewiring group of a reference run, the host LUTs,
    stats and events; plus the first steps' spikes of a free run."""
    from sparsewire.topomap import TopomapModel, formation_probability
    for (tag, scale, seed, dur, depress) in (("s1", 1, 3, 20.0, False), ("s2dep", 2, 5, 5.0, True)):
        model = TopomapModel(scale, seed)
        n = model.geometry.n
        dist = model.geometry.toroidal_distance(0, np.arange(n))
        out = {"dist": dist, "ff_lut": formation_probability(model.ff_params, dist),
               "lat_lut": formation_probability(model.lat_params, dist),
               "meta": np.array([scale, seed], dtype=np.int64)}
        if depress:
            for name in ("ff", "lat"):
                m, syn = model.net.matrices[name]
                syn.planes["g"][m.slot_mask()] = 0.05
        recs = []
        orig = model.net.run_update_group

        def wrapped(group, _orig=orig, _recs=recs, _model=model):
            pre = _tm_snap(_model)
            _orig(group)
            post = _tm_snap(_model)
            ev = {}
            for r in ("ff", "lat"):
                rule = getattr(_model, f"{r}_rule")
                ev[f"{r}_attempts"] = rule.attempts.copy()
                ev[f"{r}_ev_kind"], ev[f"{r}_ev_d"] = _tm_events(rule)
            _recs.append((pre, post, ev))
        model.net.run_update_group = wrapped
        model.run(dur)
        for k, (pre, post, ev) in enumerate(recs):
            for key, v in pre.items():
                out[f"u{k}_pre_{key}"] = v
            for key, v in post.items():
                if key.endswith("_g") or key.endswith("_target") or key.endswith("row_length"):
                    out[f"u{k}_post_{key}"] = v
            for key, v in ev.items():
                out[f"u{k}_{key}"] = v
        out["n_updates"] = np.int64(len(recs))
        save(f"topomap_{tag}.npz", **out)
    # free run: Poisson source spikes and target spikes of the first 300 steps
    model = TopomapModel(1, seed=11)
    src_log, tgt_log, pend = [], [], []
    sp, tp = model.source.poisson_step, model.target.step

    def psrc(rng, h, _f=sp):
        s_ = _f(rng, h)
        src_log.append(s_.copy())
        return s_

    def ptgt(pending, k, _f=tp):
        pend.append(pending.copy())
        t_ = _f(pending, k)
        tgt_log.append(t_.copy())
        return t_
    model.source.poisson_step = psrc
    model.target.step = ptgt
    model.run(30.0)
    st = model.state_arrays()
    src = np.zeros((len(src_log), model.geometry.n), dtype=bool)
    tgt = np.zeros_like(src)
    for t_, (a, b) in enumerate(zip(src_log, tgt_log)):
        src[t_, a] = True
        tgt[t_, b] = True
    save("topomap_run.npz", src=src, tgt=tgt, pending=np.array(pend),
         **{f"state_{k.replace('.', '_')}": v for k, v in st.items()})


def gen_stdp():
    from sparsewire.plasticity import StdpSynapses, StdpParams
    rng = R.CounterRng(12, "stdp")
    P, N, cap = 40, 30, 12
    m = RaggedMatrix(P, N, cap)
    syn = SynVarMatrix(m, ("g",))
    for i in range(P):
        k = rng.uniform_int(cap + 1)
        m.target[i, :k] = rng.sample_k_distinct(k, N)
        m.row_length[i] = k
        syn.planes["g"][i, :k] = rng.uniform01_array(k) * 0.2
    tm = TransposeMap(m)
    tm.rebuild()
    st = StdpSynapses(m, syn, 0.1, StdpParams())
    out = {"target": m.target.copy(), "row_length": m.row_length.copy(), "g0": syn.planes["g"].copy()}
    for t in range(40):
        pre = np.flatnonzero(rng.uniform01_array(P) < 0.3)
        post = np.flatnonzero(rng.uniform01_array(N) < 0.3)
        out[f"pre{t}"] = np.isin(np.arange(P), pre)
        out[f"post{t}"] = np.isin(np.arange(N), post)
        st.decay_step()
        if pre.size:
            st.on_pre_spikes(pre)
        if post.size:
            st.on_post_spikes(tm, post)
    out["g"] = syn.planes["g"].copy()
    out["x"] = st.x.copy()
    out["y"] = st.y.copy()
    save("stdp.npz", **out)


def gen_recorder():
    """TopomapRecorder CSV outputs of a short reference run (topomap.py:235-318,
    cli.py:117-125) with the edge lists of every snapshot and the rewiring
    events, so the device recorder's writers can be checked byte-for-byte on
    the same state."""
    import io
    from sparsewire.topomap import TopomapModel, TopomapRecorder
    model = TopomapModel(1, seed=6)
    rec = TopomapRecorder(snapshot_every_ms=10.0, record_spikes=True)
    states = []
    orig = rec.snapshot

    def snap(t_ms, mdl, tag=None, rows=True, _orig=orig):
        st = {"t": np.float64(t_ms), "tag": np.array(tag or ""), "rows": np.bool_(rows)}
        for proj in ("ff", "lat"):
            m, syn = mdl.net.matrices[proj]
            st[f"{proj}_row_length"] = m.row_length.copy()
            st[f"{proj}_target"] = m.target.copy()
            st[f"{proj}_g"] = syn.planes["g"].copy()
        states.append(st)
        _orig(t_ms, mdl, tag=tag, rows=rows)
    rec.snapshot = snap
    model.run(30.0, rec)
    out = {"n_states": np.int64(len(states))}
    for k, st in enumerate(states):
        for key, v in st.items():
            out[f"s{k}_{key}"] = v
    texts = {}
    for name, fn in (("degrees", rec.write_degrees_csv), ("profile", rec.write_profile_csv)):
        fh = io.StringIO()
        fn(fh)
        texts[name] = fh.getvalue()
    for kind in ("elimination", "formation"):
        fh = io.StringIO()
        rec.write_events_csv(fh, kind)
        texts[f"events_{kind}"] = fh.getvalue()
    for pop in ("source", "target"):
        fh = io.StringIO()
        rec.write_spikes_csv(fh, pop)
        texts[f"spikes_{pop}"] = fh.getvalue()
        sp = np.array(rec.spikes[pop], dtype=np.float64).reshape(-1, 2)
        out[f"spikes_{pop}"] = sp
    for (proj, kind), ev in rec.events.items():
        out[f"events_{proj}_{kind}"] = np.array(ev, dtype=np.float64).reshape(-1, 2)
    for proj in ("ff", "lat"):
        for tag in ("initial", "final"):
            pre, post, w = rec.snapshots[(proj, tag)]
            fh = io.StringIO()
            fh.write("pre,post,weight\n")
            for k in np.lexsort((post, pre)):
                fh.write(f"{pre[k]},{post[k]},{float(w[k])!r}\n")
            texts[f"connectivity_{proj}_{tag}"] = fh.getvalue()
    for k, v in texts.items():
        out[f"csv_{k}"] = np.array(v)
    save("recorder.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_recorder()
    gen_topomap()
    gen_stdp()
    gen_trainer()
    gen_rng()
    gen_remove()
    gen_deep_r()
    gen_adam()
    gen_alif_eprop()
    gen_transpose_prop()
