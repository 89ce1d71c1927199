# r02 call M (4 GPUs): weak scaling of the bench through the library NCCL exchange (config 3: N = 1, 2, 4;
# config 5: N = 4), the multi-GPU tests on 4 GPUs.
python -c "from paper_2304_05301_b200 import build; build.build()"
nvidia-smi --query-gpu=index,name,clocks.sm --format=csv
python bench.py --no-cpu-baseline --no-baselines > gpurun_out/r02m_scale_c3_n1.json 2> gpurun_out/r02m_scale_c3_n1.err
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n > gpurun_out/r02m_scale_c3_n$n.json 2> gpurun_out/r02m_scale_c3_n$n.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29549 bench.py --gpus 4 --config 5 > gpurun_out/r02m_scale_c5_n4.json 2> gpurun_out/r02m_scale_c5_n4.err
python bench.py --config 5 --no-cpu-baseline --no-baselines > gpurun_out/r02m_scale_c5_n1.json 2> gpurun_out/r02m_scale_c5_n1.err
for f in gpurun_out/r02m_scale_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d['ms_per_step'], d['e2e']['value'])"; done
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r02m_pytest_multigpu_4gpu.log 2>&1; echo "multigpu rc=$?"; tail -2 gpurun_out/r02m_pytest_multigpu_4gpu.log
