"""Envelope of Z after reverse Cuthill-McKee on the camera co-visibility graph:
bandwidth, envelope fraction, envelope-Cholesky work relative to dense.
usage: python tools/envelope_stats.py [CONFIG ...]"""
import sys; sys.path.insert(0, '.')
import numpy as np, scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee
from paper_1808_02414_b200 import synthetic as S, subrec as R
for cfg in [int(a) for a in sys.argv[1:]] or (2,3,4):
    rec = S.generate_config(cfg)
    n = rec.num_cameras()
    g = R.build_view_graph(rec)
    rows=[];cols=[]
    for a in range(n):
        for b,w in g.edges[a]: rows.append(a); cols.append(b)
    A = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n,n))
    A = A + sp.eye(n)
    nnz_frac = A.nnz / n / n
    perm = reverse_cuthill_mckee(A.tocsr(), symmetric_mode=True)
    B = A[perm][:, perm].tocoo()
    bw = np.max(np.abs(B.row - B.col))
    # profile: for each row i, first nonzero column
    first = np.full(n, n); 
    for r,c in zip(B.row,B.col): first[r]=min(first[r],c)
    prof = np.sum(np.arange(n) - first)  # lower envelope size in blocks
    # flops estimate: envelope Cholesky ~ sum over rows of (row width)^2 ; dense n^3/3 blocks
    widths = np.arange(n) - first
    chol_blocks = np.sum(widths.astype(float)**2)
    print(f"config {cfg}: n {n}, block density {nnz_frac:.3f}, RCM bandwidth {bw} cams ({bw/n:.2f} n), envelope {prof/(n*n/2):.2f} of lower triangle, env-chol work / dense {chol_blocks/(n**3/3):.3f}", flush=True)
