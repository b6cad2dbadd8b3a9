"""Scene IO (reference include/sfmcov/scene_io.hpp; tests ported from
tests/test_scene_io.cpp) plus the binary format.  CPU except the invariant
check, which runs the CUDA library's validation."""
import numpy as np
import pytest

from paper_1808_02414_b200 import sfmcov as F
from paper_1808_02414_b200 import scene_io as IO
from paper_1808_02414_b200 import synthetic as S


def same_scene(a, b):
    assert a.num_cameras() == b.num_cameras() and a.num_points() == b.num_points()
    assert a.num_observations() == b.num_observations()
    assert np.array_equal(a.cams, b.cams) and np.array_equal(a.pts, b.pts)
    assert np.array_equal(a.obs_cam, b.obs_cam) and np.array_equal(a.obs_pt, b.obs_pt)
    assert np.array_equal(a.obs_u, b.obs_u) and np.array_equal(a.obs_sigma, b.obs_sigma)


@pytest.mark.parametrize("P", [8, 9])
def test_scene_round_trips_bit_exactly(tmp_path, P):  # test_scene_io.cpp:46-69
    rec = S.generate_cube_scene(3, 0.7, P)
    p1, p2 = tmp_path / "cube.json", tmp_path / "cube2.json"
    IO.save_reconstruction(rec, p1)
    back = IO.load_reconstruction(p1, validate=False)
    same_scene(rec, back)
    IO.save_reconstruction(back, p2)  # a second save reproduces the bytes
    assert p1.read_bytes() == p2.read_bytes()


def test_identity_covariance_is_omitted(tmp_path):  # test_scene_io.cpp:71-80
    p = tmp_path / "noiseless.json"
    IO.save_reconstruction(S.generate_cube_scene(1, 0.0), p)
    assert b"sigma" not in p.read_bytes()
    back = IO.load_reconstruction(p, validate=False)
    assert np.array_equal(back.obs_sigma, np.broadcast_to(np.eye(2), back.obs_sigma.shape))
    IO.save_reconstruction(S.generate_cube_scene(1, 0.5), p)
    assert b"sigma" in p.read_bytes()


@pytest.mark.parametrize("text,fragment", [  # test_scene_io.cpp:82-96
    ("this is not json", "load"),
    ('{"points": [], "observations": []}', "cameras"),
    ('{"cameras": [{"C": [0,0,0], "c": 1, "k": 0}], "points": [], "observations": []}', "camera 0"),
    ('{"cameras": [{"r": [0,0,0], "C": [0,0,0], "c": "x", "k": 0}], "points": [], "observations": []}', "'c'"),
    ('{"cameras": [{"r": [0,0], "C": [0,0,0], "c": 1, "k": 0}], "points": [], "observations": []}', "'r'"),
    ('{"cameras": [], "points": [[0, 1]], "observations": []}', "point 0: must be an array of 3"),
    ('{"cameras": [], "points": [], "observations": [{"cam": 0, "pt": 0}]}', "observation 0: missing field 'u'"),
    ('{"cameras": 3, "points": [], "observations": []}', "top-level 'cameras' is not an array"),
])
def test_malformed_input_is_reported_with_context(tmp_path, text, fragment):
    p = tmp_path / "bad.json"
    p.write_text(text)
    with pytest.raises(F.Error) as e:
        IO.load_reconstruction(p, validate=False)
    assert e.value.kind == F.ErrorKind.parse and e.value.stage == "load"
    assert fragment in str(e.value)


def test_missing_and_unwritable_files_raise_io_errors(tmp_path):  # test_scene_io.cpp:112-125
    with pytest.raises(F.Error) as e:
        IO.load_reconstruction("/tmp/sfmcov_io_does_not_exist.json")
    assert e.value.kind == F.ErrorKind.io
    with pytest.raises(F.Error) as e:
        IO.save_reconstruction(S.generate_cube_scene(1, 0.0), "/nonexistent_dir/x.json")
    assert e.value.kind == F.ErrorKind.io


def test_saving_an_empty_reconstruction_is_rejected(tmp_path):  # test_scene_io.cpp:127-135
    empty = F.Reconstruction(np.zeros((0, 8)), np.zeros((0, 3)), np.zeros(0, np.int32), np.zeros(0, np.int32),
                             np.zeros((0, 2)), np.zeros((0, 2, 2)))
    with pytest.raises(F.Error) as e:
        IO.save_reconstruction(empty, tmp_path / "empty.json")
    assert e.value.kind == F.ErrorKind.invariant


@pytest.mark.parametrize("P", [8, 9])
def test_binary_round_trip(tmp_path, P):
    rec = S.generate_random_scene(20, 150, 0.3, 5, 0.5, P)
    p = tmp_path / "scene.bin"
    IO.save_reconstruction_binary(rec, p)
    same_scene(rec, IO.load_reconstruction_binary(p, validate=False))
    q = tmp_path / "junk.bin"
    q.write_bytes(b"not a scene")
    with pytest.raises(F.Error) as e:
        IO.load_reconstruction_binary(q, validate=False)
    assert e.value.kind == F.ErrorKind.parse


@pytest.mark.gpu
def test_load_rejects_scenes_that_violate_the_invariants(tmp_path):  # test_scene_io.cpp:98-110
    text = """{
        "cameras": [{"r": [0,0,0], "C": [0,0,-10], "c": 100, "k": 0},
                    {"r": [0,0,0], "C": [1,0,-10], "c": 100, "k": 0}],
        "points": [[0,0,0],[1,0,0],[0,1,0],[1,1,0],[0,0,1],[1,0,1],[0,1,1],[1,1,1]],
        "observations": [{"cam": 0, "pt": 0, "u": [0,0]},
                         {"cam": 1, "pt": 0, "u": [0,0]}]
    }"""
    p = tmp_path / "invalid.json"
    p.write_text(text)
    with pytest.raises(F.Error):
        IO.load_reconstruction(p)
    rec = S.generate_config(1)
    IO.save_reconstruction(rec, tmp_path / "c1.json")
    same_scene(rec, IO.load_reconstruction(tmp_path / "c1.json"))  # valid scenes pass validation
