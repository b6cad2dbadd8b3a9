# A/B of the pair-reduction kernels on config 3 (device step and stage times)
python -m pytest tests/test_gpu_parity.py -q -x -k "schur or config3_parity or golden" 2>&1 | tail -1
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('$1', round(d['value']*1e3,3), 'pair', round(s['schur_pair_reduce'],3), 'chol', round(s['cholesky'],3), 'prep', round(s['schur_point_prep'],3))"; }
SFMCOV_PAIR_KERNEL=gather run gather
for v in 2 3; do SFMCOV_PAIR_CP=$v run cp$v; done
