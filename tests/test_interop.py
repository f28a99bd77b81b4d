"""Interop with files the REFERENCE wrote.

tests/golden/interop/ holds TEALM1 / TEALW1 / TEALH1 / TEALG1 / TEALC1 files
produced by the reference's own writers (tests/golden/make_interop.py:
model.save_model, tensor.save_matrix, sparsifier.save_histogram,
greedy.save_trace / save_configs — pkg/src/actsparse/model.py:436-474,
tensor.py:197-235, sparsifier.py:189-219, greedy.py:200-271).

CPU: this package's readers load every file and its writers re-emit it
byte for byte (the `%.17g` round trip), with the values the reference
recorded.  GPU: the loaded histograms invert to the reference's thresholds
bit for bit, and the loaded model driven by the loaded TEALC1 configs
reproduces the reference's model_forward_sparse rows — through the sequence
forward and through the persistent decode engine, one position per step.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

D = GOLDEN / "interop"


def _manifest():
    return json.loads((D / "manifest.json").read_text())


def _expect():
    return np.load(D / "expect.npz")


@pytest.fixture(scope="module")
def T():
    import paper_2408_14690_b200 as T
    return T


@pytest.mark.parametrize("name,shape", [("model.teal", (2, 64, 4, 176)), ("model256.teal", (1, 256, 4, 256))])
def test_model_file_round_trip(T, tmp_path, name, shape):
    m = T.load_model(D / name)
    assert (len(m.blocks), m.d_model, m.n_heads, m.d_ff) == shape
    T.save_model(tmp_path / "m", m)
    assert (tmp_path / "m").read_bytes() == (D / name).read_bytes()


def test_matrix_file_round_trip(T, tmp_path):
    w = T.load_matrix(D / "matrix.teal")
    assert np.array_equal(w.to_2d(), _expect()["matrix"])
    assert w.layout == T.Layout.COL_MAJOR
    T.save_matrix(tmp_path / "w", w)
    assert (tmp_path / "w").read_bytes() == (D / "matrix.teal").read_bytes()


@pytest.mark.parametrize("name", _manifest()["histograms"])
def test_histogram_file_round_trip(T, tmp_path, name):
    h = T.load_histogram(D / name)
    assert h.total == int(h.counts.sum()) + h.overflow_count
    T.save_histogram(tmp_path / "h", h)
    assert (tmp_path / "h").read_bytes() == (D / name).read_bytes()


def test_trace_file_round_trip(T, tmp_path):
    tr = T.load_trace(D / "trace.txt")
    assert [s.block_sparsity for s in tr.steps] == _expect()["trace_P"].tolist()
    T.save_trace(tmp_path / "t", tr)
    assert (tmp_path / "t").read_bytes() == (D / "trace.txt").read_bytes()


def test_config_file_round_trip(T, tmp_path):
    cfgs, target = T.load_configs(D / "configs.txt")
    e = _expect()
    names = ("q", "k", "v", "o", "gate", "up", "down")
    assert target == 0.5 and len(cfgs) == 2
    assert [[c.thresholds[n] for n in names] for c in cfgs] == e["cfg_thresholds"].tolist()
    assert [[c.levels[n] for n in names] for c in cfgs] == e["cfg_levels"].tolist()
    T.save_configs(tmp_path / "c", cfgs, target)
    assert (tmp_path / "c").read_bytes() == (D / "configs.txt").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", _manifest()["histograms"])
def test_reference_histograms_invert_bit_exact(T, name):
    h = T.load_histogram(D / name)
    e = _expect()
    assert h.thresholds(e["p_grid"]) == e[f"thr_{name}"].tolist()


@pytest.mark.gpu
def test_reference_model_and_configs_drive_the_gpu_forward(T):
    m = T.load_model(D / "model.teal")
    cfgs, _ = T.load_configs(D / "configs.txt")
    e = _expect()
    out = T.model_forward_sparse(m, e["X"], cfgs)
    out = out.cpu().numpy() if hasattr(out, "cpu") else np.asarray(out)
    assert rel_err(out, e["out_sparse"]) < 1e-5
    dense = T.model_forward_dense(m, e["X"])
    dense = dense.cpu().numpy() if hasattr(dense, "cpu") else np.asarray(dense)
    assert rel_err(dense, e["out_dense"]) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["step", "launch"])
def test_reference_configs_drive_the_decode_engines(T, engine):
    # the decode step at position t equals row t of the reference's forward
    # (causality, pkg/tests/test_model.py:171-178), thresholds from TEALC1
    from paper_2408_14690_b200 import decode as Dm
    from paper_2408_14690_b200 import engine as E
    from paper_2408_14690_b200.model import decoder_weights
    # the step engine tiles d, n_q in multiples of 256: its run uses the
    # one-block d = 256 model and its reference-written TEALC1 file
    sfx = "256" if engine == "step" else ""
    m = T.load_model(D / f"model{sfx}.teal")
    cfgs, _ = T.load_configs(D / f"configs{sfx}.txt")
    e = _expect()
    X, want = e[f"X{sfx}"], e[f"out{sfx}_sparse"]
    thr = [[c.thresholds[n] for n in Dm.PROJ] for c in cfgs]
    W = decoder_weights(m, max_seq=16)
    dec = E.StepDecoder(W, thr) if engine == "step" else Dm.SparseDecoder(W, thr)
    dec.reset()
    errs = [rel_err(dec.step_hidden(X[t]).cpu().numpy(), want[t]) for t in range(len(X))]
    assert np.median(errs) < 1e-5 and max(errs) < 1e-4, (np.median(errs), max(errs))
