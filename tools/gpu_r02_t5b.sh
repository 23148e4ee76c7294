# A/B after the instruction diet: the ticketed kernel at 5 CTAs/SM (48 registers) vs 4, N=2
set -x
O=gpurun_out/r02t5b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/t5.so GTC_TICKET_CTAS=5 >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000"
p=29600
for rho in 0.01 0.1; do for i in 1 2; do
p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_t4_${rho}_$i.jsonl 2> /dev/null
p=$((p+1)); GTC_LIB=/tmp/t5.so timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_t5_${rho}_$i.jsonl 2> /dev/null
done; done
