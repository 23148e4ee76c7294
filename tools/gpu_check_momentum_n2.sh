# 2-GPU: the fused step in GTC_ACCUM_MOMENTUM mode (parity + bench) and the
# fused vs separate-kernel step at 10 % density
set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "fused_step_parity and momentum" > gpurun_out/mgpu2_mom.log 2>&1; echo mgpu=$?
tail -3 gpurun_out/mgpu2_mom.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 2 --steps 300 --warmup 10 --no-e2e"
timeout 300 $B --accum momentum > gpurun_out/bench_n2_mom.jsonl 2> gpurun_out/bench_n2_mom.err
GTC_STEP_FUSED=0 timeout 300 $B --accum momentum > gpurun_out/bench_n2_mom_unfused.jsonl 2>/dev/null
timeout 300 $B --rho 0.1 > gpurun_out/bench_n2_rho10.jsonl 2>/dev/null
GTC_STEP_FUSED=0 timeout 300 $B --rho 0.1 > gpurun_out/bench_n2_rho10_unfused.jsonl 2>/dev/null
timeout 300 $B --rho 0.001 > gpurun_out/bench_n2_rho01.jsonl 2>/dev/null
GTC_DECODE_TRACE=1 TRACE_TAIL=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py > gpurun_out/trace_n2.txt 2>&1
