"""Fresh-engine first-call check (device path, flush, profiling) — race hunt."""
import sys, os, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, _native as N
mode = sys.argv[1]
rec = S.generate_config(3)
dev = torch.device("cuda", 0)
tens = {k: torch.from_numpy(getattr(rec, k)).to(dev) for k in ("cams", "pts", "obs_cam", "obs_pt", "obs_u", "obs_sigma")}
P, n = rec.cam_params, rec.num_cameras()
sc = N.Scene(); sc.n_cams, sc.n_pts, sc.n_obs, sc.cam_params = n, rec.num_points(), rec.num_observations(), P
sc.cams, sc.pts = tens["cams"].data_ptr(), tens["pts"].data_ptr()
sc.obs_cam, sc.obs_pt = tens["obs_cam"].data_ptr(), tens["obs_pt"].data_ptr()
sc.obs_u, sc.obs_sigma = tens["obs_u"].data_ptr(), tens["obs_sigma"].data_ptr()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
torch.cuda.synchronize()
lib = N.cuda_lib()
opts = N.Options(0, 0, 0, 0); diag = N.Diagnostics(); err = N.ErrorStruct()
bad = 0
for trial in range(int(sys.argv[2])):
    eng = F.Engine(0)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    d_cov = torch.empty((n, P, P), dtype=torch.float64, device=dev)
    eng.set_profiling('p' in mode)
    for it in range(2):
        if 'f' in mode:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
        code = lib.sfmcov_cuda_compute_covariance_device(eng.handle, C.byref(sc), C.byref(opts), d_cov.data_ptr(), C.byref(diag), C.byref(err))
        if code:
            bad += 1; print(trial, it, "ERROR", err.message.decode(), flush=True)
    eng.close()
print(mode, "bad", bad, flush=True)
