# 4-GPU check of the fused p2p step: parity tests at world 3/4, bench lines
# (fused vs separate kernels)
set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "fused or (exchange_parity and p2p and gt)" > gpurun_out/mgpu4.log 2>&1; echo mgpu=$?
tail -3 gpurun_out/mgpu4.log
GTC_DECODE_TRACE=1 TRACE_TAIL=4 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py > gpurun_out/trace_n4.txt 2>&1
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --steps 300 --warmup 10 --no-e2e"
timeout 300 $B > gpurun_out/bench_n4.jsonl 2> gpurun_out/bench_n4.err; echo b4=$?
GTC_STEP_FUSED=0 timeout 300 $B > gpurun_out/bench_n4_unfused.jsonl 2>/dev/null
