# phase trace of the final fused step at N=2, and the 0.01 % density line
GTC_DECODE_TRACE=1 TRACE_TAIL=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py > gpurun_out/trace_n2_final.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 2 --steps 300 --warmup 10 --no-e2e --rho 0.0001 > gpurun_out/bench_n2_rho001.jsonl 2>/dev/null
