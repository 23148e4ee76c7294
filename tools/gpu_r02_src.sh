# ncu source-level capture (instructions and stall samples per line) of the N=1 step kernel and of the
# ticketed N>1 kernel (world-2 loopback group), one launch each
set -x
O=gpurun_out/r02src2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B --steps 300 --warmup 5 > $O/plain.jsonl 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_encode_tile_kernel -s 200 -c 1 -o $O/n1 $B --steps 300 --warmup 5 > $O/ncu_n1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_step_ticket_group -s 30 -c 1 -o $O/lb2 python tools/loopback_bench.py --world 2 --steps 40 > $O/ncu_lb2.log 2>&1
