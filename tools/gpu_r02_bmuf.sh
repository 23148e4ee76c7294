# final tree: BMUF (the paper's second trainer) lines at N = 1, 2, 4
set -x
O=gpurun_out/r02bmuf; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --algo bmuf --no-e2e --no-cpu-baseline > $O/bench_n1_bmuf.jsonl 2> $O/e1
p=29990
for N in 2 4; do
  p=$((p+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $p bench.py --gpus $N --algo bmuf --no-e2e > $O/bench_n${N}_bmuf.jsonl 2> $O/e$N
done
