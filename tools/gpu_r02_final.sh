# round 2 final tree (ticketed kernel at 5 CTAs/SM): N = 1, 2, 4 bench lines on one 4-GPU box, the full
set -x
O=${O:-gpurun_out/r02fin}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/e_n1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --rho 0.1 > $O/bench_n1_rho10.jsonl 2> $O/e_n1r
timeout 600 python bench.py --no-cpu-baseline --no-e2e --accum momentum > $O/bench_n1_mom.jsonl 2> $O/e_n1m
timeout 900 python bench.py --workload 1e9 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_n1_1e9.jsonl 2> $O/e_n1g
p=29800
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  p=$((p+1)); timeout 600 $TR --master-port $p bench.py --gpus $N > $O/bench_n${N}.jsonl 2> $O/e_n$N
  p=$((p+1)); timeout 600 $TR --master-port $p bench.py --gpus $N --no-e2e --rho 0.1 > $O/bench_n${N}_rho10.jsonl 2> $O/e_n${N}r
  p=$((p+1)); timeout 600 $TR --master-port $p bench.py --gpus $N --no-e2e --accum momentum > $O/bench_n${N}_mom.jsonl 2> $O/e_n${N}m
  p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus $N --workload 1e9 --steps 20 --warmup 3 --no-e2e > $O/bench_n${N}_1e9.jsonl 2> $O/e_n${N}g
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "EXIT $?" >> $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu_4gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu_4gpu.log
