# One GPU, the round's evidence: GPU suite + smoke, the bounds-checked build on the sanitize cases
# (compute-sanitizer is closed on the pool), bench lines (config 3 default + reference arm, configs
# 2, 4, 4 x 64 seeds, 5), e2e breakdown, launch list + full ncu of config 3's and config 4's search.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2304_05301_b200 import build; build.build()"
python paper_2304_05301_b200/build.py --variant checked -DTACOS_CHECKED=1 > /dev/null
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
TACOS_LIB=paper_2304_05301_b200/libtacos_checked.so python tools/sanitize_cases.py > gpurun_out/checked_cases.txt 2>&1; tail -1 gpurun_out/checked_cases.txt
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json | cut -c1-400
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_c3.json 2>&1
python bench.py --config 2 --no-baselines > gpurun_out/bench_c2.json 2>&1
python bench.py --config 5 --no-baselines > gpurun_out/bench_c5.json 2>&1
python bench.py --config 4 --steps 5 --warmup 3 --e2e-steps 2 --no-baselines > gpurun_out/bench_c4.json 2>&1
python bench.py --config 4 --seeds 64 --steps 3 --warmup 3 --e2e-steps 1 --no-baselines --no-cpu-baseline > gpurun_out/bench_c4_s64.json 2>&1
python bench.py --literal --no-baselines > gpurun_out/bench_c3_literal.json 2>&1
python bench.py --config 6 --no-baselines > gpurun_out/bench_ctx.json 2>&1
python tools/host_breakdown.py 3 > gpurun_out/e2e_breakdown_c3.txt 2>&1
python tools/trace_windows.py 4 > gpurun_out/trace_windows_c4_summary.txt 2>&1
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-baselines --e2e-steps 1"
python bench.py $ARGS > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy -s 3 -c 1 -o gpurun_out/prof_c3 -f python bench.py $ARGS > gpurun_out/ncu_c3.log 2>&1
python tools/time_search.py 4 0 1 > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/prof_c4 -f python tools/time_search.py 4 0 1 > gpurun_out/ncu_c4.log 2>&1
# then, here: python tools/make_profiles.py rNN c3_torus8x8x8_ar gpurun_out/launches_c3.csv gpurun_out/prof_c3.ncu-rep
