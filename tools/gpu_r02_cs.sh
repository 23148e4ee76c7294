# A/B on one GPU: evict-first (.cs) loads/stores of the r/g stream vs L1::no_allocate (default), N=1
set -x
O=gpurun_out/r02cs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/cs.so GTC_STREAM_CS >> $O/build.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 2000"
for i in 1 2; do
timeout 300 $B > $O/bench_def_$i.jsonl 2>/dev/null
GTC_LIB=/tmp/cs.so timeout 300 $B > $O/bench_cs_$i.jsonl 2>/dev/null
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline --rho 0.1 > $O/bench_def_rho10.jsonl 2>/dev/null
GTC_LIB=/tmp/cs.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --rho 0.1 > $O/bench_cs_rho10.jsonl 2>/dev/null
