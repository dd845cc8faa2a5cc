"""Matrix Market ingestion and CSR validation: the product's
host reader/writer/validators against the reference's golden behaviour
(tests/golden/mm_cases.json, from oracle/make_mm_golden.py) and, where the
reference library is built, against it directly on large generated files
(several parse chunks, shuffled entries, errors placed in late chunks).
CPU only -- ingestion is host code feeding the device upload."""
import json
import os

import numpy as np
import pytest

import paper_2603_09790_b200 as cs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mm_cases.json")))
CODES = {1: cs.DimensionError, 2: cs.InvalidMatrixError, 3: cs.NotSpdError, 7: cs.ParseError}


def _write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def _vals(hexes):
    return np.array([float.fromhex(v) for v in hexes])


@pytest.mark.parametrize("case", GOLD["read"], ids=lambda c: c["name"])
def test_read_matches_reference(tmp_path, case):
    path = _write(tmp_path, case["text"])
    exp = case["expect"]
    if "error" in exp:
        with pytest.raises(CODES[exp["error"]["code"]]) as ei:
            cs.read_matrix_market(path, case["require_spd"])
        assert str(ei.value) == exp["error"]["msg"].replace("<path>", path)
        assert type(ei.value) is CODES[exp["error"]["code"]]
        return
    a = cs.read_matrix_market(path, case["require_spd"])
    ok = exp["ok"]
    assert a.n == ok["n"]
    assert a.row_offsets.tolist() == ok["rowptr"]
    assert a.col_indices.tolist() == ok["col"]
    assert a.values.tobytes() == _vals(ok["val_hex"]).tobytes()


def test_missing_file(tmp_path):
    p = str(tmp_path / "nope.mtx")
    with pytest.raises(cs.ParseError, match="cannot open " + p):
        cs.read_matrix_market(p)


@pytest.mark.parametrize("case", GOLD["validate"], ids=lambda c: c["name"])
def test_validate_matches_reference(case):
    c = case["csr"]
    a = cs.CsrMatrix(c["n"], np.array(c["rowptr"]), np.array(c["col"]), _vals(c["val_hex"]))
    fns = {"0": cs.validate_structure, "1": cs.validate_symmetric, "2": cs.validate_spd_diagonal}
    for k, exp in case["expect"].items():
        if exp is None:
            fns[k](a)
        else:
            with pytest.raises(CODES[exp["code"]]) as ei:
                fns[k](a)
            assert str(ei.value) == exp["msg"]


def test_write_matches_reference(tmp_path):
    w = GOLD["write"][0]
    c = w["csr"]
    a = cs.CsrMatrix(c["n"], np.array(c["rowptr"]), np.array(c["col"]), _vals(c["val_hex"]))
    p = str(tmp_path / "w.mtx")
    cs.write_matrix_market(p, a)
    assert open(p).read() == w["text"]


def _random_spd_text(rng, n, extra_per_row, *, crlf=False, shuffle=True):
    """symmetric, strictly diagonally dominant; lower-triangle entries in random order"""
    rows, cols = [], []
    for i in range(n):
        js = rng.choice(n, size=extra_per_row, replace=False)
        for j in js:
            if j < i:
                rows.append(i)
                cols.append(j)
    pairs = np.unique(np.array([rows, cols]).T, axis=0) if rows else np.zeros((0, 2), int)
    off = -rng.random(len(pairs))
    lines = [f"{i + 1} {j + 1} {float(v)!r}" for (i, j), v in zip(pairs, off)]
    lines += [f"{i + 1} {i + 1} {float(2 * extra_per_row + 1 + rng.random())!r}" for i in range(n)]
    if shuffle:
        rng.shuffle(lines)
    nl = "\r\n" if crlf else "\n"
    body = nl.join(lines)
    return (f"%%MatrixMarket matrix coordinate real symmetric{nl}% generated{nl}"
            f"{n} {n} {len(lines)}{nl}{body}{nl}"), len(lines)


def test_large_random_files_match_reference(tmp_path, ref):
    rng = np.random.default_rng(11)
    for k, (n, e, crlf) in enumerate([(3000, 9, False), (20000, 7, True)]):
        text, _ = _random_spd_text(rng, n, e, crlf=crlf)
        assert len(text) > 1 << 17  # several parse chunks
        path = _write(tmp_path, text, f"r{k}.mtx")
        a = cs.read_matrix_market(path, True)
        r = ref.mm_read(path, True)
        assert a.row_offsets.tobytes() == r.rowptr.tobytes()
        assert a.col_indices.tobytes() == r.col.tobytes()
        assert a.values.tobytes() == r.val.tobytes()
        cs.validate_symmetric(a)
        # writer round trip is byte-identical to the reference writer
        p1, p2 = str(tmp_path / "o1.mtx"), str(tmp_path / "o2.mtx")
        cs.write_matrix_market(p1, a)
        ref.mm_write(p2, r)
        assert open(p1, "rb").read() == open(p2, "rb").read()
        b = cs.read_matrix_market(p1, True)
        assert b.values.tobytes() == a.values.tobytes()


@pytest.mark.parametrize("where", ["late_error", "late_fewer", "garbage_tail", "dup_late"])
def test_large_file_errors_match_reference(tmp_path, ref, where):
    rng = np.random.default_rng(5)
    text, count = _random_spd_text(rng, 8000, 6)
    lines = text.split("\n")
    if where == "late_error":
        lines[-50] = "12 x 0.5"
    elif where == "late_fewer":
        lines[2] = lines[2].rsplit(" ", 1)[0] + f" {count + 3}"
    elif where == "garbage_tail":
        lines = lines[:-1] + ["not an entry", "1 1 nan", ""]
    elif where == "dup_late":
        lines[-2] = lines[5]
    path = _write(tmp_path, "\n".join(lines))
    try:
        r = ref.mm_read(path, True)
        ref_err = None
    except Exception as e:  # OracleError
        ref_err = (e.code, e.msg)
    if ref_err is None:
        a = cs.read_matrix_market(path, True)
        assert a.col_indices.tobytes() == r.col.tobytes()
        assert a.values.tobytes() == r.val.tobytes()
    else:
        with pytest.raises(CODES[ref_err[0]]) as ei:
            cs.read_matrix_market(path, True)
        assert str(ei.value) == ref_err[1]


def test_csr_host_rows_block(tmp_path):
    rng = np.random.default_rng(3)
    text, _ = _random_spd_text(rng, 500, 5)
    path = _write(tmp_path, text)
    a = cs.read_matrix_market(path)
    # row blocks of the partition reassemble the matrix
    parts = [cs.partition_rows(a.n, 1, 3, r) for r in range(3)]
    assert parts[0][0] == 0 and parts[-1][1] == a.n
    for b, e in parts:
        rp = a.row_offsets[b:e + 1] - a.row_offsets[b]
        assert rp[0] == 0 and rp[-1] == a.row_offsets[e] - a.row_offsets[b]
