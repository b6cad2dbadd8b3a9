"""Scene IO (reference include/sfmcov/scene_io.hpp): the reference's JSON
format (bit-exact round trip) and a binary format for large scenes.
Host library (libsfmcov_synth.so); loading validates the scene's invariants
through the CUDA library unless validate=False."""
from __future__ import annotations

import ctypes as C

from . import _native as N
from .sfmcov import Error, Reconstruction, _raise
from .synthetic import _take


def _load(fn, path: str, validate: bool) -> Reconstruction:
    err = N.ErrorStruct()
    h = fn(str(path).encode(), C.byref(err))
    if not h:
        raise Error(err.kind, err.stage.decode(), err.message.decode())
    rec = _take(h)
    if validate:
        rec.validate()
    return rec


def load_reconstruction(path: str, validate: bool = True) -> Reconstruction:
    return _load(N.synth_lib().sfmcov_scene_load, path, validate)


def save_reconstruction(rec: Reconstruction, path: str) -> None:
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.synth_lib().sfmcov_scene_save(C.byref(sc), str(path).encode(), C.byref(err)), err)


def load_reconstruction_binary(path: str, validate: bool = True) -> Reconstruction:
    return _load(N.synth_lib().sfmcov_scene_load_binary, path, validate)


def save_reconstruction_binary(rec: Reconstruction, path: str) -> None:
    err = N.ErrorStruct()
    sc = rec.c_struct()
    _raise(N.synth_lib().sfmcov_scene_save_binary(C.byref(sc), str(path).encode(), C.byref(err)), err)
