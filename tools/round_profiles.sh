# The round's evidence on one B200 (outputs under gpurun_out/, copied to
# profiles/ by hand): bench lines for configs 3 (with the CPU baseline), 4, 5,
# the reference arm, the config-3 ncu launch list with DRAM bytes, the
# sub-reconstruction throughput.
set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c3.log 2>&1
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv --sweep > gpurun_out/launches_c3.txt 2>&1
python tools/subrec_bench.py 3 > gpurun_out/subrec_c3.log 2>&1
