# N GPUs (gpurun --gpus N): the multi-GPU tests, then weak scaling of the bench through the library's
# NCCL exchange (torchrun, one process per GPU): config 3 at 1, 2, N GPUs and config 5 at 1 and N.
N=${N:-4}
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_multigpu.log 2>&1; tail -1 gpurun_out/pytest_multigpu.log
for cfg in 3 5; do
  for n in 1 2 $N; do
    [ $cfg = 5 ] && [ $n = 2 ] && continue
    if [ $n = 1 ]; then python bench.py --config $cfg --no-cpu-baseline --no-baselines > gpurun_out/scale_c${cfg}_n1.json 2>&1;
    else python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 295$cfg$n \
         bench.py --gpus $n --config $cfg > gpurun_out/scale_c${cfg}_n$n.json 2> gpurun_out/scale_c${cfg}_n$n.err; fi
    tail -1 gpurun_out/scale_c${cfg}_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($cfg, $n, d['value'], d['ms_per_step'])"
  done
done
