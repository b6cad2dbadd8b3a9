"""Dense-stage time of one big config for the current SFMCOV_PANEL (profiling aid)."""
import os, sys
sys.path.insert(0, '.')
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
cfg = int(sys.argv[1])
rec = S.generate_config(cfg)
eng = F.Engine(0)
eng.set_profiling(True)
for it in range(2):
    eng.compute_covariance(rec)
    st = eng.stage_times()
    print(f"config {cfg} panel {os.environ.get('SFMCOV_PANEL', 'auto')} run {it}: cholesky {st['cholesky']:.1f} ms", flush=True)
