"""Covariance IO (reference src/covariance_io.cpp:17-122; the file shapes the
reference's tests/test_cli.cpp:98-127 checks).  Host library only: CPU tests,
plus one GPU round trip of a real result."""
import json

import numpy as np
import pytest

from paper_1808_02414_b200 import covariance_io as IO
from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import synthetic as S


def random_result(n, P, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, P, P))
    cov = np.einsum("nij,nkj->nik", a, a) * 10.0 ** rng.integers(-9, 3, (n, 1, 1))
    diag = F.CovarianceDiagnostics(scale_min=1.25e-5, scale_max=3.0, flagged_columns=[3, 17], min_pivot=0.0017,
                                   max_pivot=12.5, inertia_positive=P * n, inertia_negative=7,
                                   negative_eigenvalue_warnings=0, peak_dense_bytes=8 * (P * n + 7) ** 2,
                                   largest_dense_dim=P * n + 7)
    return F.CovarianceResult(cov, diag)


@pytest.mark.parametrize("P", [8, 9])
def test_pack_upper_triangle_order_and_round_trip(P):  # covariance_io.hpp:10-13
    m = np.arange(P * P, dtype=float).reshape(P, P)
    m = m + m.T
    tri = IO.pack_upper_triangle(m)
    assert len(tri) == P * (P + 1) // 2
    assert np.array_equal(tri, np.concatenate([m[r, r:] for r in range(P)]))
    assert np.array_equal(IO.unpack_upper_triangle(tri), m)


@pytest.mark.parametrize("P", [8, 9])
def test_json_is_the_reference_dump_and_round_trips(tmp_path, P):
    res = random_result(6, P)
    path = tmp_path / "cov.json"
    IO.save_covariance_json(res, path)
    text = path.read_text()
    doc = json.loads(text)
    assert len(doc["cameras"]) == 6 and all(len(c["cov"]) == P * (P + 1) // 2 for c in doc["cameras"])
    assert [c["id"] for c in doc["cameras"]] == list(range(6))
    assert doc["diagnostics"]["inertia_negative"] == 7 and doc["diagnostics"]["flagged_columns"] == [3, 17]
    # nlohmann::json::dump(): sorted keys, compact separators, shortest round-trip doubles
    assert text == json.dumps(doc, separators=(",", ":"), sort_keys=True) + "\n"
    back = IO.load_covariance_json(path, P)
    assert np.array_equal(back.camera_cov, res.camera_cov)  # bit-exact
    assert back.diagnostics == res.diagnostics


def test_csv_header_rows_and_precision(tmp_path):  # test_cli.cpp:116-126
    res = random_result(6, 8, 1)
    path = tmp_path / "cov.csv"
    IO.save_covariance_csv(res, path)
    lines = path.read_text().splitlines()
    assert lines[0].startswith("id,cov_0_0") and lines[0].count(",") == 36
    assert len(lines) == 7
    for i, line in enumerate(lines[1:]):
        cells = line.split(",")
        assert int(cells[0]) == i
        assert np.array_equal(np.array([float(c) for c in cells[1:]]), IO.pack_upper_triangle(res.camera_cov[i]))


def test_load_errors(tmp_path):
    with pytest.raises(F.Error) as e:
        IO.load_covariance_json(tmp_path / "missing.json")
    assert e.value.kind == F.ErrorKind.io
    bad = tmp_path / "bad.json"
    bad.write_text("this is not json")
    with pytest.raises(F.Error) as e:
        IO.load_covariance_json(bad)
    assert e.value.kind == F.ErrorKind.parse and e.value.stage == "load"
    bad.write_text('{"cameras":[{"cov":[1,2],"id":0}],"diagnostics":{}}')
    with pytest.raises(F.Error) as e:
        IO.load_covariance_json(bad)
    assert e.value.kind == F.ErrorKind.parse and "bad covariance file" in str(e.value)
    with pytest.raises(F.Error) as e:
        IO.save_covariance_json(random_result(2, 8), tmp_path / "no_such_dir" / "x.json")
    assert e.value.kind == F.ErrorKind.io and e.value.stage == "save"


@pytest.mark.gpu
def test_gpu_result_round_trip(engine, tmp_path):  # test_cli.cpp:98-113
    res = engine.compute_covariance(S.generate_cube_scene(3, 0.5))
    IO.save_covariance_json(res, tmp_path / "cov.json")
    back = IO.load_covariance_json(tmp_path / "cov.json")
    # the file holds the upper triangle (the blocks are symmetric to the last bit,
    # not bitwise, in the reference too: (s_p Z_pq) s_q vs (s_q Z_qp) s_p)
    for a, b in zip(back.camera_cov, res.camera_cov):
        assert np.array_equal(IO.pack_upper_triangle(a), IO.pack_upper_triangle(b))
        assert np.abs(a - b).max() <= 1e-15 * np.abs(b).max()
    assert back.diagnostics == res.diagnostics and back.diagnostics.inertia_negative == 7
