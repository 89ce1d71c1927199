# r02 call R (2 GPUs): device-resident winner for the emission -- full GPU suite incl. multi-GPU, bench.
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests -m gpu -x -q > gpurun_out/r02r_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02r_pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 python bench.py --no-baselines > gpurun_out/r02r_bench_c3.json 2> gpurun_out/r02r_bench_c3.err; tail -c 300 gpurun_out/r02r_bench_c3.json
CUDA_VISIBLE_DEVICES=0 python tools/host_breakdown.py 3 > gpurun_out/r02r_host_breakdown_c3.txt 2>&1; cat gpurun_out/r02r_host_breakdown_c3.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/r02r_bench_c3_n2.json 2> gpurun_out/r02r_bench_c3_n2.err; tail -c 200 gpurun_out/r02r_bench_c3_n2.json
