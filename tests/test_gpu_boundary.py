"""GPU: the drop-in's on-disk and concurrency contracts.

* SSSD v1 files written from a GPU-built datastore are byte-identical to the
  reference writer's (ref datastore.py:11-19,220-226; golden sha256 / bytes in
  tests/golden/files.json made by tests/golden/make_golden.py from the
  reference itself), through ``Datastore.save`` and the ``build-datastore``
  CLI (ref cli.py:37-47); reference-written bytes load back and re-save equal.
* Concurrent proposes from several host threads (each with its own stream,
  workspace and outputs; "unbounded concurrent readers") give
  the drafts of a serial run, bit for bit."""

import hashlib
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2411_05894_b200 as G  # noqa: E402
from paper_2411_05894_b200 import workload  # noqa: E402
from paper_2411_05894_b200.cli import main as cli_main  # noqa: E402


def _corpus(rec):
    if "corpus" in rec:
        return rec["corpus"]
    n, v = (int(x) for x in rec["workload"][len("corpus("):-1].split(","))
    return workload.corpus(n, v).tolist()


def test_saved_file_is_byte_identical_to_reference(golden, tmp_path):
    for rec in golden("files.json"):
        corpus = _corpus(rec)
        path = tmp_path / "ds.bin"
        G.build(corpus, vocab_size=rec["vocab"]).save(path)
        data = path.read_bytes()
        assert len(data) == rec["bytes"] and hashlib.sha256(data).hexdigest() == rec["sha256"]
        if "hex" in rec:  # reference-written bytes load and re-save unchanged
            src = tmp_path / "ref.bin"
            src.write_bytes(bytes.fromhex(rec["hex"]))
            ds = G.load(src)
            assert ds.tokens.tolist() == corpus
            ds.save(tmp_path / "again.bin")
            assert (tmp_path / "again.bin").read_bytes() == bytes.fromhex(rec["hex"])


def test_cli_build_datastore_bytes(golden, tmp_path):
    rec = [r for r in golden("files.json") if r.get("workload", "").startswith("corpus(50000")][0]
    corpus = np.asarray(_corpus(rec), dtype="<u4")
    tok = tmp_path / "c.tok"
    corpus.tofile(tok)
    out = tmp_path / "cli.bin"
    assert cli_main(["build-datastore", "--in", str(tok), "--out", str(out), "--vocab-size", "1000"]) == 0
    assert hashlib.sha256(out.read_bytes()).hexdigest() == rec["sha256"]


def test_concurrent_host_threads_propose_bit_identical():
    corpus = workload.corpus(500_000, 2000)
    ds = G.build(corpus, vocab_size=2000)
    eng = G.DraftEngine(ds, G.FusionConfig(dec_len=32))
    T, B = 4, 96
    batches = []
    for t in range(T):
        ctxs = workload.contexts(B, 300, 2000, seed=40 + t)
        seq, off, ln, mx = eng.upload([c.tolist() for c in ctxs])
        want = eng.propose(seq, off, ln, mx)
        want = {k: getattr(want, k).clone() for k in ("size", "tokens", "parents", "depths", "mask")}
        batches.append((seq, off, ln, mx, want))
    eng.check_status()
    torch.cuda.synchronize()
    errs = []

    def worker(t):
        try:
            seq, off, ln, mx, want = batches[t]
            st = torch.cuda.Stream()
            ws = torch.empty(eng.workspace(B, mx).numel(), dtype=torch.uint8, device="cuda")
            out = eng.new_outputs(B)
            for _ in range(5):
                eng.propose(seq, off, ln, mx, out=out, ws=ws, stream=st)
                st.synchronize()
                for k, v in want.items():
                    g = getattr(out, k)
                    if k == "size":
                        assert torch.equal(g, v)
                    else:
                        for b in range(B):
                            n = int(want["size"][b])
                            assert torch.equal(g[b, :n], v[b, :n]), (t, k, b)
        except Exception as exc:  # surfaced below
            errs.append(repr(exc))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(T)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs


def test_sa_check_accepts_the_index_and_catches_corruption():
    rng = np.random.default_rng(9)
    for n, alpha in ((1, 3), (7, 2), (5000, 3), (200_000, 50)):
        corpus = rng.integers(0, alpha, n).astype(np.uint32)
        ds = G.build(corpus)
        rep = ds.check()
        assert rep["ok"] and rep["adjacent_not_increasing"] == 0 and rep["positions_missing"] == 0, (n, rep)
    rows = ds.rows
    a, b = 1000, 1001
    tmp = rows[a].clone()
    rows[a] = rows[b]
    rows[b] = tmp
    rep = ds.check()
    assert not rep["ok"] and rep["adjacent_not_increasing"] >= 1
    rows[b] = rows[a]  # duplicate position -> one missing
    rep = ds.check()
    assert rep["positions_missing"] == 1
