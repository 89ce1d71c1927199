# r02 call L: final 1-GPU bench lines (config 3 default + reference arm, configs 2, 4, 4x64, 5), launch list + full ncu of config 3.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2304_05301_b200 import build; build.build()"
python bench.py > gpurun_out/r02l_bench_c3.json 2> gpurun_out/r02l_bench_c3.err; tail -c 300 gpurun_out/r02l_bench_c3.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02l_bench_ref_c3.json 2>&1; tail -c 300 gpurun_out/r02l_bench_ref_c3.json
python bench.py --config 2 --no-baselines > gpurun_out/r02l_bench_c2.json 2>&1; tail -c 200 gpurun_out/r02l_bench_c2.json
python bench.py --config 5 --no-baselines > gpurun_out/r02l_bench_c5.json 2>&1; tail -c 200 gpurun_out/r02l_bench_c5.json
python bench.py --config 4 --steps 5 --warmup 3 --e2e-steps 2 --no-baselines > gpurun_out/r02l_bench_c4.json 2>&1; tail -c 200 gpurun_out/r02l_bench_c4.json
python bench.py --config 4 --seeds 64 --steps 3 --warmup 3 --e2e-steps 1 --no-baselines --no-cpu-baseline > gpurun_out/r02l_bench_c4_s64.json 2>&1; tail -c 200 gpurun_out/r02l_bench_c4_s64.json
python tools/host_breakdown.py 3 > gpurun_out/r02l_host_breakdown_c3.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 1 > gpurun_out/r02l_plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_launches_c3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 1 > gpurun_out/r02l_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy -s 3 -c 1 -o gpurun_out/r02l_prof_c3 -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 1 > gpurun_out/r02l_ncu_full.log 2>&1; echo "ncu rc=$?"
