# Round-end ncu evidence on one B200 (after the same command has exited 0 without ncu):
# --set full captures of the two bulk GEMM classes of the config-3 sweep (the first
# Cholesky trailing update and a mid-sweep inverse "rows below" update), summarised by
# tools/ncu_summary.py; the per-camera truth table of the final code; the sweep trace.
set -x
mkdir -p gpurun_out
python tools/sweep_components.py 3 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:k_gemm<\(bool\)0, \(int\)16, \(int\)3, \(int\)64, \(int\)64' --launch-skip 7 --launch-count 1 -f -o gpurun_out/ncu_gemm_tri \
    python tools/sweep_components.py 3 > gpurun_out/ncu_gemm_tri.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:k_gemm<\(bool\)1, \(int\)16, \(int\)3, \(int\)64, \(int\)64' --launch-skip 35 --launch-count 1 -f -o gpurun_out/ncu_gemm_inv \
    python tools/sweep_components.py 3 > gpurun_out/ncu_gemm_inv.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_gemm_tri.ncu-rep > gpurun_out/ncu_gemm_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/ncu_gemm_inv.ncu-rep >> gpurun_out/ncu_gemm_summary.txt 2>&1
SFMCOV_SWEEP_TRACE=1 python tools/sweep_components.py 3 2> gpurun_out/trace_c3.txt
python tools/trace_view.py gpurun_out/trace_c3.txt --chain > gpurun_out/trace_c3_view.txt 2>&1
python tools/truth_gpu.py cube small c1 c2 c3 readme c4 > gpurun_out/truth_final.log 2>&1
python tools/truth_gpu.py c5 --sample 48 >> gpurun_out/truth_final.log 2>&1
