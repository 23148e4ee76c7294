set -x
O=gpurun_out/r02w7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/loopback_bench.py --world 2 --steps 30 > $O/lb2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_step_ws_group -s 20 -c 1 -o $O/ws_lb2 python tools/loopback_bench.py --world 2 --steps 30 > $O/ncu.log 2>&1
