# 4-GPU: every multi-GPU parity test (fused step incl. momentum, split step,
# NCCL, BMUF) and the momentum bench at N=4, fused vs split
set -x
mkdir -p gpurun_out/n4
timeout 1200 python -m pytest tests/test_multigpu.py -q > gpurun_out/n4/pytest_multigpu_4gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/n4/pytest_multigpu_4gpu.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --steps 300 --warmup 10 --no-e2e --accum momentum"
timeout 300 $B > gpurun_out/n4/bench_n4_mom.jsonl 2> gpurun_out/n4/bench_n4_mom.err
timeout 300 $B --split-step > gpurun_out/n4/bench_n4_mom_split.jsonl 2>/dev/null
