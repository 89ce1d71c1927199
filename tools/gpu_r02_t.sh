# r02 call T: bench lines with the final roofline fields (configs 3, 4, 4 x 64, 5, 2).
python -c "from paper_2304_05301_b200 import build; build.build()"
python bench.py > gpurun_out/r02t_bench_c3.json 2>&1
python bench.py --config 4 --steps 5 --warmup 3 --e2e-steps 2 --no-baselines > gpurun_out/r02t_bench_c4.json 2>&1
python bench.py --config 4 --seeds 64 --steps 3 --warmup 3 --e2e-steps 1 --no-baselines --no-cpu-baseline > gpurun_out/r02t_bench_c4_s64.json 2>&1
python bench.py --config 5 --no-baselines > gpurun_out/r02t_bench_c5.json 2>&1
python bench.py --config 2 --no-baselines > gpurun_out/r02t_bench_c2.json 2>&1
for f in c3 c4 c4_s64 c5 c2; do tail -c 200 gpurun_out/r02t_bench_$f.json; echo; done
