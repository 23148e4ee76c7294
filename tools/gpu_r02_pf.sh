# A/B: L2 prefetch of a dense tile's target lines before the overflow round (GTC_TARGET_PREFETCH) at N=2
set -x
O=gpurun_out/r02pf; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/nopf.so GTC_TARGET_PREFETCH=0 >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000"
p=30100
for rep in 1 2; do
for rho in 0.1 0.01; do
  p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_n2_r${rho}_pf_$rep.jsonl 2> /dev/null
  p=$((p+1)); GTC_LIB=/tmp/nopf.so timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_n2_r${rho}_nopf_$rep.jsonl 2> /dev/null
done
done
timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
