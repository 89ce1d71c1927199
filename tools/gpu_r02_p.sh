# r02 call P: new parity tests (CUSTOM windowed, large FC), bench default line with the final bench.py.
python -c "from paper_2304_05301_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "custom_pre_post or large_fully" > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02p_pytest.log
python bench.py > gpurun_out/r02p_bench_c3.json 2> gpurun_out/r02p_bench_c3.err; tail -c 400 gpurun_out/r02p_bench_c3.json
