#!/bin/bash
# round-2 GPU pass AZ: the N > 1 bench path at HEAD (2 ranks, gloo, both on the one GPU: functional, not a performance number)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_az.log 2>&1
RS_TRACE_SHARDED=1 RS_BENCH_BACKEND=gloo RS_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C2 --steps 3 --warmup 3 > gpurun_out/bench_gloo2_az.json 2> gpurun_out/bench_gloo2_az.err; echo "rc=$?" >> gpurun_out/bench_gloo2_az.err
echo done
