export PCCL_TIMEOUT_MS=8000
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"; tail -5 gpurun_out/gpu_tests.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29640"
for np in 2 4; do
 for ll in 0 1048576; do
  PCCL_LL_MAX=$ll timeout 300 $T --nproc-per-node $np tools/latency.py --sizes 16384,262144,1048576,2097152,4194304 --algos direct --no-nccl 2>&1 | grep "p=" | sed "s/^/ll_max=$ll /"
 done
done
