"""One fresh process, first call on a config: report whether the dense stage needed a serial retry."""
import sys
sys.path.insert(0, '.')
from paper_1808_02414_b200 import synthetic as S, sfmcov as F
rec = S.generate_config(int(sys.argv[1]))
eng = F.Engine(0)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    eng.compute_covariance(rec)
    print("call", i, "retries", eng.counts()["dense_retries"], flush=True)
