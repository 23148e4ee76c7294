# A/B on one GPU: the world-1 step kernel at 4 / 5 / 6 CTAs per SM (64 / 48 / 40 registers)
set -x
O=gpurun_out/r02enc5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/e5.so GTC_ENC_CTAS=5 >> $O/build.log 2>&1 &
python tools/build_variant.py /tmp/e6.so GTC_ENC_CTAS=6 >> $O/build.log 2>&1 &
wait
B="python bench.py --no-e2e --no-cpu-baseline --steps 2000"
for i in 1 2; do
timeout 300 $B > $O/bench_e4_$i.jsonl 2>/dev/null
GTC_LIB=/tmp/e5.so timeout 300 $B > $O/bench_e5_$i.jsonl 2>/dev/null
GTC_LIB=/tmp/e6.so timeout 300 $B > $O/bench_e6_$i.jsonl 2>/dev/null
done
