# Emulated multi-GPU sweeps with per-component timing (SFMCOV_DIST_TRACE=1),
# replayed on R GPUs by tools/dist_schedule.py.
mkdir -p gpurun_out
for cr in "3 8" "4 1" "4 2" "4 4" "4 8" "5 8"; do
  set -- $cr
  SFMCOV_DIST_TRACE=1 timeout 1500 python tools/dist_schedule.py run $1 $2 2> gpurun_out/dtrace_c$1_r$2.txt
  echo "== config $1, R = $2"
  python tools/dist_schedule.py read gpurun_out/dtrace_c$1_r$2.txt
done
