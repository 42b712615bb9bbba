# the N>1 code path of bench.py on one GPU (torchrun, world 1, NCCL)
BENCH_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 1 --steps 300 --warmup 5 --cpu-seconds 2 --no-c3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
echo rc=$?; tail -5 gpurun_out/bench_dist1.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_dist1.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d.get('c4'))"
