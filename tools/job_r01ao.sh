#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "
import torch
from paper_2411_18424_b200.dataplane import host_link_info, numa_nodes
print(host_link_info('cuda:0'), numa_nodes())"
nvidia-smi topo -m 2>&1 | head -12
KVS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 2 --warmup 3 --no-sweep --no-trace > gpurun_out/bench_ao2.json 2> gpurun_out/bench_ao2.err; tail -2 gpurun_out/bench_ao2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_ao2.json').read().strip().splitlines()[-1])
print(json.dumps(d['roofline']['aggregate']), json.dumps(d['roofline']['host_links']), d['config']['host_pool'])"
