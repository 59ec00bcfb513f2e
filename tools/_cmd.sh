export PCCL_TIMEOUT_MS=8000
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29620"
timeout 300 $T tools/probe.py --pats a2a,uni --modes 0,1,2,3 --ctas 16,32,64,128,256 2>&1 | grep "p=4" > gpurun_out/probe256.log
cat gpurun_out/probe256.log
timeout 400 $T tools/tune.py --size-mib 128 --ctas 16,32,64,128 --algos direct --variants 1,2,3 --colls ag_f32 --tma 4x32768,3x65536,8x16384,2x98304 2>&1 | grep "p=4" > gpurun_out/tune_tma.log
cat gpurun_out/tune_tma.log
