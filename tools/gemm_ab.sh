# A/B of the DMMA shape in k_gemm (SFMCOV_GEMM_MMA=16 | 4): the fragment-layout
# probe, the dense parity tests, then config 3 / 4 steps for both shapes.
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/dmma16 tools/probe/dmma16_layout.cu && /tmp/dmma16
python -m pytest tests/test_gpu_parity.py tests/test_gpu_truth.py -q -x -k "config3 or camera_covariance or truth or wide_dense or spd" 2>&1 | tail -1
run() { python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 config $2', round(d['value']*1e3,3), 'chol', round(d['stages_ms']['cholesky'],3), 'frac', round(d['roofline']['frac'],4))"; }
for r in 1 2; do for m in 4 16; do SFMCOV_GEMM_MMA=$m run mma$m 3 10; done; done
for m in 4 16; do SFMCOV_GEMM_MMA=$m run mma$m 4 3; done
