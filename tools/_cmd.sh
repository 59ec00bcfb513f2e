export PCCL_TIMEOUT_MS=8000
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29640"
timeout 300 $T --nproc-per-node 2 tools/latency.py --sizes 16384,1048576 --algos direct --no-nccl --api python 2>&1 | grep "p=\|Error\|error" | head
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -p no:cacheprovider 2>&1 | tail -3
