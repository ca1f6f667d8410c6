"""TopomapRecorder (topomap.py:235-318, cli.py:117-125) on the device model:
the writers must reproduce the reference's CSV bytes for the same state.

CPU: the snapshot statistics and every writer, fed the reference run's own
edge lists, events and spikes (tests/golden/recorder.npz, made by
make_golden.py from the real reference).  GPU: the same snapshots taken from
a device TopomapModel whose connectivity is injected from those states, and
a recorder run of the device model end to end."""

import io

import numpy as np
import pytest

from conftest import golden


def _states(d):
    out = []
    for k in range(int(d["n_states"])):
        out.append({key[len(f"s{k}_"):]: d[key] for key in d.files if key.startswith(f"s{k}_")})
    return out


def _edges(st, proj):
    rl, tg, g = st[f"{proj}_row_length"], st[f"{proj}_target"], st[f"{proj}_g"]
    mask = np.arange(tg.shape[1])[None, :] < rl[:, None]
    pre = np.repeat(np.arange(len(rl), dtype=np.int64), rl.astype(np.int64))
    return pre, tg[mask].astype(np.int64), g[mask], rl


def _texts(rec):
    out = {}
    for name, fn in (("degrees", rec.write_degrees_csv), ("profile", rec.write_profile_csv)):
        fh = io.StringIO()
        fn(fh)
        out[name] = fh.getvalue()
    for kind in ("elimination", "formation"):
        fh = io.StringIO()
        rec.write_events_csv(fh, kind)
        out[f"events_{kind}"] = fh.getvalue()
    for pop in ("source", "target"):
        fh = io.StringIO()
        rec.write_spikes_csv(fh, pop)
        out[f"spikes_{pop}"] = fh.getvalue()
    for proj in ("ff", "lat"):
        for tag in ("initial", "final"):
            fh = io.StringIO()
            rec.write_connectivity_csv(fh, proj, tag)
            out[f"connectivity_{proj}_{tag}"] = fh.getvalue()
    return out


def _fill_events_spikes(rec, d):
    for proj in ("ff", "lat"):
        for kind in ("elimination", "formation"):
            rec.events[(proj, kind)] = [tuple(x) for x in d[f"events_{proj}_{kind}"].tolist()]
    for pop in ("source", "target"):
        for t, i in d[f"spikes_{pop}"].tolist():
            rec.on_spikes(pop, t, [int(i)])


def test_recorder_writers_byte_identical_host():
    from paper_2510_19764_b200.geometry import GridGeometry
    from paper_2510_19764_b200.topomap import TopomapRecorder
    d = golden("recorder.npz")
    geom = GridGeometry(16)
    rec = TopomapRecorder(snapshot_every_ms=10.0, record_spikes=True)
    for st in _states(d):
        tag = str(st["tag"]) or None
        for proj in ("ff", "lat"):
            pre, post, w, rl = _edges(st, proj)
            rec.snapshot_edges(float(st["t"]), proj, geom, pre, post, w, rl, geom.n,
                               tag=tag, rows=bool(st["rows"]))
    _fill_events_spikes(rec, d)
    got = _texts(rec)
    for k, v in got.items():
        assert v == str(d[f"csv_{k}"]), k
    assert got["events_formation"].count("\n") > 1 and got["spikes_source"].count("\n") > 10


@pytest.mark.gpu
def test_recorder_device_snapshots_byte_identical(dev_lib):
    from paper_2510_19764_b200.topomap import TopomapModel, TopomapRecorder
    d = golden("recorder.npz")
    model = TopomapModel(1, seed=6, use_graph=False)
    rec = TopomapRecorder(snapshot_every_ms=10.0, record_spikes=True)
    for st in _states(d):
        for proj in ("ff", "lat"):
            m, syn = model.net.matrices[proj]
            rl, tg, g = st[f"{proj}_row_length"], st[f"{proj}_target"], st[f"{proj}_g"]
            assert tg.shape[1] == m.stride
            m.load_state(rl, tg)
            syn.planes["g"].copy_(__import__("torch").from_numpy(np.ascontiguousarray(g)))
        rec.snapshot(float(st["t"]), model, tag=str(st["tag"]) or None, rows=bool(st["rows"]))
    _fill_events_spikes(rec, d)
    got = _texts(rec)
    for k, v in got.items():
        assert v == str(d[f"csv_{k}"]), k


@pytest.mark.gpu
def test_recorder_device_run(dev_lib):
    """A device run with a recorder: snapshots every 10 ms, spikes and events
    recorded, the final edge lists equal the model's state."""
    from paper_2510_19764_b200.topomap import TopomapModel, TopomapRecorder
    model = TopomapModel(1, seed=6)
    rec = TopomapRecorder(snapshot_every_ms=10.0, record_spikes=True)
    model.run(30.0, rec)
    t = _texts(rec)
    assert t["degrees"].count("\n") == 1 + 2 * 4          # 0, 10, 20, 30 ms x 2 projections
    assert t["profile"].count("\n") == 1 + 2 * 4 * 16
    assert t["spikes_source"].count("\n") > 10
    pre, post, w, rl, n = TopomapRecorder.host_edges(model, "ff")
    fp, fq, fw = rec.snapshots[("ff", "final")]
    assert np.array_equal(pre, fp) and np.array_equal(post, fq) and np.array_equal(w, fw)
    assert sum(len(v) for v in rec.events.values()) > 0
    # graph path (no spikes, no events): snapshots between replays
    model2 = TopomapModel(1, seed=6, record_events=False)
    rec2 = TopomapRecorder(snapshot_every_ms=10.0)
    model2.run(30.0, rec2)
    assert len(rec2.degrees) == 2 * 4
