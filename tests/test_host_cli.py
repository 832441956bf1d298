"""C++ host API / CLI (include/gsr/cuda_api.hpp, tools/gsrnet_cuda.cpp) and the
graph-store binary formats."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2603_27156_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "gsrnet-cuda")


@pytest.fixture(scope="module")
def cli():
    from paper_2603_27156_b200 import build
    build.build()
    return CLI


def _files(tmp_path, n=400, seed=0):
    g, nd = synth.generate_synthetic(synth.SynthConfig(n=n, hub_fraction=0.01, hub_degree_range=(10, 40), seed=seed))
    gp, np_ = str(tmp_path / "g.gsrg"), str(tmp_path / "n.gsrn")
    synth.write_graph(gp, g)
    synth.write_node_data(np_, nd)
    return g, nd, gp, np_


def test_gsrg_gsrn_round_trip(tmp_path):
    g, nd, gp, np_ = _files(tmp_path)
    g2 = synth.read_graph(gp)
    nd2 = synth.read_node_data(np_)
    assert g2.n == g.n and np.array_equal(g2.row_ptr, g.row_ptr) and np.array_equal(g2.col_idx, g.col_idx)
    assert np.array_equal(nd2.features, nd.features) and np.array_equal(nd2.labels, nd.labels)
    assert np.array_equal(nd2.split, nd.split)


def test_gsrg_rejects_corruption(tmp_path):
    _, _, gp, np_ = _files(tmp_path)
    b = bytearray(open(gp, "rb").read())
    open(gp, "wb").write(b[:-3])
    with pytest.raises(ValueError, match="truncated"):
        synth.read_graph(gp)
    b[0:4] = b"XXXX"
    open(gp, "wb").write(b)
    with pytest.raises(ValueError, match="magic"):
        synth.read_graph(gp)


def test_gsrp_round_trip_and_corruption(tmp_path):
    from paper_2603_27156_b200 import MODE_GSRC, model
    p = model.init_params(MODE_GSRC, 3, 64, 4, 8, seed=4)
    path = str(tmp_path / "p.gsrp")
    model.write_gsrp(path, p, MODE_GSRC, 3, 64, 4, 8)
    q, meta = model.read_gsrp(path)
    assert np.array_equal(p, q) and meta == dict(mode=MODE_GSRC, layers=3, hidden=64, groups=4, d_in=8)
    b = open(path, "rb").read()
    open(path, "wb").write(b[:-8])
    with pytest.raises(ValueError, match="truncated"):
        model.read_gsrp(path)
    open(path, "wb").write(b"GSRX" + b[4:])
    with pytest.raises(ValueError, match="magic"):
        model.read_gsrp(path)


def test_cli_exit_codes_without_gpu(cli, tmp_path):
    _, _, gp, np_ = _files(tmp_path)
    r = subprocess.run([cli, "version"], capture_output=True, text=True)
    assert r.returncode == 0 and "gsrnet 0.1.0" in r.stdout
    r = subprocess.run([cli, "train", "--graph", str(tmp_path / "missing.gsrg"), "--nodes", np_], capture_output=True, text=True)
    assert r.returncode == 3, r.stderr        # ResourceError → exit 3
    r = subprocess.run([cli, "train", "--graph", gp, "--nodes", np_, "--model", "bogus"], capture_output=True, text=True)
    assert r.returncode == 1, r.stderr        # ConfigError → exit 1
    bad = tmp_path / "bad.gsrg"
    bad.write_bytes(b"NOPE" + b"\0" * 40)
    r = subprocess.run([cli, "train", "--graph", str(bad), "--nodes", np_], capture_output=True, text=True)
    assert r.returncode == 1 and "magic" in r.stderr   # FormatError is a ConfigError


@pytest.mark.gpu
def test_cli_trains_and_matches_python_host(cli, tmp_path):
    """Same graph, node file and initial params through the C++ host and the
    Python host: identical first-epoch loss (both run the same C-ABI)."""
    from paper_2603_27156_b200 import MODE_GSRC, Context, init_params
    g, nd, gp, np_ = _files(tmp_path, n=2000)
    L, D, C, k = 3, 64, 2, 8
    p = init_params(MODE_GSRC, L, D, C, 8, seed=3)
    pf = tmp_path / "p.f32"
    p.astype(np.float32).tofile(pf)
    rep = tmp_path / "r.jsonl"
    r = subprocess.run([cli, "train", "--graph", gp, "--nodes", np_, "--layers", str(L), "--hidden", str(D), "--groups", str(C),
                        "--k", str(k), "--epochs", "4", "--lr", "1e-3", "--params", str(pf), "--report", str(rep)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    recs = [json.loads(x) for x in rep.read_text().splitlines()]
    assert [x["record"] for x in recs] == ["epoch"] * 4 + ["metrics", "summary"]
    assert recs[-1]["kernel_launches"] > 0
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(MODE_GSRC, L, D, C, k, 8)
    ctx.set_params(p)
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    losses = [ctx.train_step(lr=1e-3) for _ in range(4)]
    assert [r["train_loss"] for r in recs[:4]] == pytest.approx(losses, rel=1e-6)
    assert recs[3]["train_loss"] < recs[0]["train_loss"]
    # Eq. 9 breakdown per epoch
    for r in recs[:4]:
        parts = r["t_forward"] + r["t_backward"] + r["t_optimizer"] + r["t_copy"]
        assert r["t_forward"] > 0 and r["t_backward"] > 0 and parts <= r["t_total"] * 1.001 + 1e-6
    # CorrelationReport per split on the final predictions
    from scipy import stats
    yhat = ctx.forward().astype(np.float64)
    met = recs[4]
    for code, name in enumerate(("train", "val", "test")):
        sel = nd.split == code
        a, b = yhat[sel], nd.labels[sel].astype(np.float64)
        m = met[name]
        assert m["count"] == int(sel.sum())
        assert m["pearson"] == pytest.approx(stats.pearsonr(a, b)[0], abs=1e-6)
        assert m["spearman"] == pytest.approx(stats.spearmanr(a, b)[0], abs=1e-6)
        assert m["kendall"] == pytest.approx(stats.kendalltau(a, b)[0], abs=1e-6)
        assert m["r2"] == pytest.approx(1 - ((b - a) ** 2).sum() / ((b - b.mean()) ** 2).sum(), abs=1e-6)


@pytest.mark.gpu
def test_cli_checkpoint_resume(cli, tmp_path):
    """--checkpoint writes GSRP of the trained parameters plus the
    Adam state sidecar (<out>.adam: m, v, step); 2 epochs + --resume 2 epochs
    equal 4 straight epochs bit for bit."""
    from paper_2603_27156_b200 import MODE_GSRC, Context, init_params, model
    g, nd, gp, np_ = _files(tmp_path, n=2000)
    L, D, C, k = 2, 64, 2, 8
    p = init_params(MODE_GSRC, L, D, C, 8, seed=5)
    pf = tmp_path / "p.f32"
    p.astype(np.float32).tofile(pf)
    ck = tmp_path / "a.gsrp"
    args = ["--graph", gp, "--nodes", np_, "--layers", str(L), "--hidden", str(D), "--groups", str(C), "--k", str(k), "--lr", "1e-3"]
    r = subprocess.run([cli, "train", *args, "--epochs", "2", "--params", str(pf), "--checkpoint", str(ck), "--report", str(tmp_path / "a.jsonl")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    q, meta = model.read_gsrp(str(ck))
    assert meta == dict(mode=MODE_GSRC, layers=L, hidden=D, groups=C, d_in=8)
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=1)
    ctx.model_init(MODE_GSRC, L, D, C, k, 8)
    ctx.set_params(p)
    ctx.data_upload(nd.features, nd.labels, nd.train_mask)
    for _ in range(2):
        ctx.train_step(lr=1e-3)
    assert np.array_equal(ctx.params(), q)
    m, v, step = ctx.optim_state()
    raw = (tmp_path / "a.gsrp.adam").read_bytes()
    assert raw[:4] == b"GSRA" and int(np.frombuffer(raw[16:24], np.int64)[0]) == step == 2
    assert np.array_equal(np.frombuffer(raw[24:24 + 4 * m.size], np.float32), m)
    ck2 = tmp_path / "b.gsrp"
    r = subprocess.run([cli, "train", *args, "--epochs", "2", "--resume", str(ck), "--checkpoint", str(ck2), "--report", str(tmp_path / "b.jsonl")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert json.loads((tmp_path / "b.jsonl").read_text().splitlines()[-1])["exact_resume"] is True
    for _ in range(2):
        ctx.train_step(lr=1e-3)
    assert np.array_equal(model.read_gsrp(str(ck2))[0], ctx.params())   # exact resume
    r = subprocess.run([cli, "train", *args[:4], "--hidden", "32", *args[6:], "--epochs", "1", "--resume", str(ck)], capture_output=True, text=True)
    assert r.returncode == 1 and "differs" in r.stderr
