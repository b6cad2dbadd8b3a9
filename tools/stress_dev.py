"""Device-path stress (torch-resident scene), optional L2 flush, like bench.py:
every call must succeed and be bitwise identical to the first.
usage: python tools/stress_dev.py FLUSH(0/1) REPS PROFILING(0/1)"""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1808_02414_b200 import synthetic as S, sfmcov as F, _native as N
flush_on = int(sys.argv[1]); reps = int(sys.argv[2]); prof = int(sys.argv[3])
rec = S.generate_config(3)
eng = F.Engine(0); lib = N.cuda_lib()
ref = eng.compute_covariance(rec).camera_cov
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(eng.stream, device=dev)
tens = {k: torch.from_numpy(getattr(rec, k)).to(dev) for k in ("cams", "pts", "obs_cam", "obs_pt", "obs_u", "obs_sigma")}
P, n = rec.cam_params, rec.num_cameras()
d_cov = torch.empty((n, P, P), dtype=torch.float64, device=dev)
sc = N.Scene(); sc.n_cams, sc.n_pts, sc.n_obs, sc.cam_params = n, rec.num_points(), rec.num_observations(), P
sc.cams, sc.pts = tens["cams"].data_ptr(), tens["pts"].data_ptr()
sc.obs_cam, sc.obs_pt = tens["obs_cam"].data_ptr(), tens["obs_pt"].data_ptr()
sc.obs_u, sc.obs_sigma = tens["obs_u"].data_ptr(), tens["obs_sigma"].data_ptr()
torch.cuda.synchronize()
opts = N.Options(0, 0, 0, 0); diag = N.Diagnostics(); err = N.ErrorStruct()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
eng.set_profiling(bool(prof))
bad = 0
for i in range(reps):
    if flush_on:
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
    code = lib.sfmcov_cuda_compute_covariance_device(eng.handle, C.byref(sc), C.byref(opts), d_cov.data_ptr(), C.byref(diag), C.byref(err))
    if code:
        bad += 1; print(i, "ERROR", err.message.decode(), flush=True); continue
    c = d_cov.cpu().numpy()
    if not np.array_equal(c, ref):
        bad += 1; print(i, "DIFF", np.abs(c - ref).max(), flush=True)
print("flush", flush_on, "prof", prof, "bad", bad, "of", reps, flush=True)
