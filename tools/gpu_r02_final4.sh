# round 2 final 4-GPU lines: 1e9-parameter workload at N = 1, 2, 4; momentum and BMUF at N = 4
set -x
O=gpurun_out/r02final4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --workload 1e9 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_n1_1e9.jsonl 2> $O/e1
p=29700
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  p=$((p+1)); timeout 900 $TR --master-port $p bench.py --gpus $N --workload 1e9 --steps 20 --warmup 3 --no-e2e > $O/bench_n${N}_1e9.jsonl 2> $O/e_1e9_$N
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29711 bench.py --gpus 4 --accum momentum --no-e2e > $O/bench_n4_mom.jsonl 2> $O/e_mom4
timeout 600 $TR --master-port 29712 bench.py --gpus 4 --algo bmuf --no-e2e > $O/bench_n4_bmuf.jsonl 2> $O/e_bmuf4
