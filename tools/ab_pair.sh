# A/B of the pair-reduction kernels on config 3 (cp: the kept cp.async kernel;
# gather: the round-1 register-gather kernel): parity subset, device step and
# stage times, then the pair kernels' own durations (ncu launch list).
python -m pytest tests/test_gpu_parity.py -q -x -k "schur or config3 or golden" 2>&1 | tail -1
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('$1', round(d['value']*1e3,3), 'pair', round(s['schur_pair_reduce'],3), 'chol', round(s['cholesky'],3), 'prep', round(s['schur_point_prep'],3))"; }
ncu_pair() { ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:k_pair_reduce -c 2 --csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import csv,sys,collections; rows=[r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=rows[0]; t=collections.defaultdict(float)
for r in rows[1:]:
    d=dict(zip(h,r)); t[d['Metric Name']]+=float(d['Metric Value'].replace(',',''))
print('$1 ncu', dict(t))"; }
for k in cp gather; do SFMCOV_PAIR_KERNEL=$k run $k; done
for k in cp gather; do SFMCOV_PAIR_KERNEL=$k ncu_pair $k; done
