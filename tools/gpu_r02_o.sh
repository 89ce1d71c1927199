# r02 call O: full GPU suite (incl. random windowed parity), smoke, config-4 bench lines with the touched
# bytes, ncu of the final config-4 kernel at 16 and 64 seeds (the latter spills L2).
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r02o_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02o_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02o_smoke.log
python bench.py --config 4 --steps 5 --warmup 3 --e2e-steps 2 --no-baselines --no-cpu-baseline > gpurun_out/r02o_bench_c4.json 2>&1; tail -c 300 gpurun_out/r02o_bench_c4.json
python bench.py --config 4 --seeds 64 --steps 3 --warmup 3 --e2e-steps 1 --no-baselines --no-cpu-baseline > gpurun_out/r02o_bench_c4_s64.json 2>&1; tail -c 300 gpurun_out/r02o_bench_c4_s64.json
python tools/time_search.py 4 0 1 > gpurun_out/r02o_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/r02o_prof_c4 -f \
    python tools/time_search.py 4 0 1 > gpurun_out/r02o_ncu_c4.log 2>&1; echo "ncu16 rc=$?"
python tools/time_search.py 4 0 1 64 > gpurun_out/r02o_c4s64_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:greedy -c 1 -o gpurun_out/r02o_prof_c4s64 -f \
    python tools/time_search.py 4 0 1 64 > gpurun_out/r02o_ncu_c4s64.log 2>&1; echo "ncu64 rc=$?"
