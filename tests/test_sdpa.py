"""SDPA reader against the reference parser's outputs.

Fixture ``tests/golden/sdpa.npz`` (make_sdpa_goldens.py, run against the live
reference): our own random / hand-written SDPA texts, valid and malformed,
with the reference's parsed entries, error type, line and message, and its
decomposition of the valid random problems.  CPU only: the reader is host
C++ in libhsde.so.
"""
import io

import numpy as np
import pytest

from paper_1611_01828_b200 import DuplicateEntry, ParseError, decompose, parse_sdpa


def _cases(golden_dir):
    z = np.load(golden_dir / "sdpa.npz")
    for t in range(int(z["n_cases"])):
        pre = f"c{t}_"
        yield z, pre, z[pre + "label"].item().decode(), z[pre + "text"].tobytes().decode()


def _table(p):
    mat, blk, i, j, v = p.entry_table
    return np.stack([mat, blk, i, j, v], axis=1).astype(float).reshape(-1, 5)


def test_parse_matches_reference(golden_dir):
    n_ok = n_err = 0
    for z, pre, label, text in _cases(golden_dir):
        kind = int(z[pre + "kind"])
        if kind == 0:
            p = parse_sdpa(text)
            assert p.m == int(z[pre + "m"]), label
            assert p.block_dims == tuple(int(d) for d in z[pre + "dims"]), label
            assert np.array_equal(p.b, z[pre + "b"]), label
            ref = z[pre + "entries"]
            got = _table(p)
            assert got.shape == ref.shape, label
            # values bit-exact (inf / -0.0 included)
            assert np.array_equal(got[:, :4], ref[:, :4]), label
            assert np.array_equal(got[:, 4].view(np.int64), ref[:, 4].view(np.int64)), label
            n_ok += 1
        else:
            exc = DuplicateEntry if kind == 2 else ParseError
            with pytest.raises(exc) as err:
                parse_sdpa(text)
            assert type(err.value) is exc, label
            assert err.value.line == int(z[pre + "line"]), label
            assert str(err.value) == z[pre + "msg"].item().decode(), label
            n_err += 1
    assert n_ok >= 10 and n_err >= 20


def test_decompose_of_parsed_matches_reference(golden_dir):
    n = 0
    for z, pre, label, text in _cases(golden_dir):
        if pre + "dec" not in z:
            continue
        cp = decompose(parse_sdpa(text))
        assert np.array_equal(cp.covered, z[pre + "covered"]), label
        assert np.array_equal(cp.c, z[pre + "c"]), label
        assert np.array_equal(cp.A.indptr, z[pre + "A_indptr"]), label
        assert np.array_equal(cp.A.indices, z[pre + "A_indices"]), label
        assert np.array_equal(cp.A.data, z[pre + "A_data"]), label
        assert np.array_equal(cp.sizes, z[pre + "clique_sizes"]), label
        assert np.array_equal(np.concatenate(cp.cliques), z[pre + "clique_nodes"]), label
        n += 1
    assert n >= 5


def test_object_view_and_fast_path_agree(golden_dir):
    """decompose() on the flat entry arrays == on the per-block SymMatrix view."""
    from types import SimpleNamespace
    for z, pre, label, text in _cases(golden_dir):
        if pre + "dec" not in z:
            continue
        p = parse_sdpa(text)
        view = SimpleNamespace(m=p.m, block_dims=p.block_dims, b=p.b, C=p.C, A=p.A)
        a, b = decompose(p), decompose(view)
        assert np.array_equal(a.covered, b.covered) and np.array_equal(a.c, b.c)
        assert (a.A != b.A).nnz == 0


def test_input_kinds_and_object_view(tmp_path):
    text = "2\n2\n{2, -3}\n1.0, 2.0\n0 1 1 2 5.0\n1 2 3 3 1.0\n2 1 2 1 -4.0\n"
    f = tmp_path / "tiny.dat-s"
    f.write_text(text)
    for src in (text, text.encode(), f, io.StringIO(text), io.BytesIO(text.encode())):
        p = parse_sdpa(src)
        assert p.m == 2 and p.block_dims == (2, -3) and p.block_sizes == (2, 3)
        assert p.n_total == 5 and p.block_offsets == (0, 2, 5) and p.entry_count() == 3
        assert p.C[0].get(1, 0) == 5.0 and p.A[0][1].get(2, 2) == 1.0
        assert p.A[1][0].entries == ((0, 1, -4.0),)
        assert np.array_equal(p.A[1][0].to_dense(), [[0.0, -4.0], [-4.0, 0.0]])


def test_large_file_round_trip():
    """10^5 entries: the C++ reader keeps every entry, sorted, i <= j."""
    rng = np.random.default_rng(5)
    m, d, ne = 50, 400, 100_000
    iu = np.triu_indices(d)
    pick = rng.choice(iu[0].size, size=ne // (m + 1), replace=False)
    lines = [f"{m}", "1", f"{d}", " ".join("1.0" for _ in range(m))]
    want = []
    for mat in range(m + 1):
        for k in pick:
            i, j = int(iu[0][k]), int(iu[1][k])
            v = float(mat + 1) + int(k) * 1e-6
            a, b = (j, i) if (k + mat) % 3 == 0 else (i, j)
            lines.append(f"{mat} 1 {a + 1} {b + 1} {v!r}")
            want.append((mat, 0, i, j, v))
    p = parse_sdpa("\n".join(lines))
    want.sort()
    assert p.entry_count() == len(want)
    assert np.array_equal(_table(p), np.asarray(want, dtype=float))
