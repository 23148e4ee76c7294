# 2-GPU check of the fused p2p step: parity tests, a phase trace, then bench
# lines (N=2 at several decode lags, and the unfused step for comparison)
set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "fused or unfused or lstm" > gpurun_out/mgpu2.log 2>&1; echo mgpu=$?
tail -3 gpurun_out/mgpu2.log
GTC_DECODE_TRACE=1 TRACE_TAIL=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py > gpurun_out/trace_n2.txt 2>&1
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 2 --steps 300 --warmup 10 --no-e2e"
timeout 300 $B > gpurun_out/bench_n2.jsonl 2> gpurun_out/bench_n2.err; echo b2=$?
for L in 1184; do GTC_FUSED_LAG=$L timeout 300 $B > gpurun_out/bench_n2_lag$L.jsonl 2>/dev/null; done
