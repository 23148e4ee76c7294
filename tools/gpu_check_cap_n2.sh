# 2-GPU: fused step with the 50 % push cap at 10 % and 1 % density
set -x
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "test_fused_step_parity and not 4- and not 3-" > gpurun_out/mgpu2_cap.log 2>&1; echo mgpu=$?
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 2 --steps 300 --warmup 10 --no-e2e"
timeout 300 $B --rho 0.1 > gpurun_out/bench_n2_rho10_cap.jsonl 2>/dev/null
timeout 300 $B > gpurun_out/bench_n2_cap.jsonl 2>/dev/null
GTC_DECODE_TRACE=1 TRACE_TAIL=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py > gpurun_out/trace_n2.txt 2>&1
