# bisection of the fused p2p step's cost at N=2 (GTC_FUSED_DIAG bits; timing only)
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 2 --steps 300 --warmup 10 --no-e2e"
for D in 0 1 3 7; do GTC_FUSED_DIAG=$D timeout 300 $B > gpurun_out/diag_$D.jsonl 2>/dev/null; done
GTC_FUSED_DIAG=7 GTC_FUSED_LAG=5930 timeout 300 $B > gpurun_out/diag_7_lagT.jsonl 2>/dev/null
