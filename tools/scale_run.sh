# N-GPU scaling of the default bench (config 3, 64 seeds per GPU), then config 5 (256 seeds sharded) at N.
N=${N:-4}
for n in 1 2 $N; do
  if [ $n = 1 ]; then python bench.py --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err;
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err; fi
  tail -1 gpurun_out/scale_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $N --config 5 --seeds $((256 / N)) --no-baselines > gpurun_out/c5_n$N.json 2> gpurun_out/c5_n$N.err
tail -1 gpurun_out/c5_n$N.json | cut -c1-400
