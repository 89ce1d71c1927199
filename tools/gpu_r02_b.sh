# r02 call B (2 GPUs): multi-GPU tests, 2-rank bench through the library's NCCL exchange, full 1-GPU suite.
nvidia-smi --query-gpu=index,name --format=csv
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests/test_multigpu.py -x -q --durations=10 > gpurun_out/r02b_pytest_multigpu.log 2>&1; echo "multigpu rc=$?"; tail -15 gpurun_out/r02b_pytest_multigpu.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02b_bench_n2.json 2> gpurun_out/r02b_bench_n2.err; echo "bench2 rc=$?"; tail -c 600 gpurun_out/r02b_bench_n2.json; tail -5 gpurun_out/r02b_bench_n2.err
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r02b_pytest_gpu.log
