# r02 call S: async emission test, bench default line.
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests/test_gpu_parity.py -x -q -k "emit_async or sharded_plans or synthesize_into or config_parity" > gpurun_out/r02s_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02s_pytest.log
python bench.py > gpurun_out/r02s_bench_c3.json 2> gpurun_out/r02s_bench_c3.err; tail -c 300 gpurun_out/r02s_bench_c3.json
