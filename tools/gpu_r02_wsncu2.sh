set -x
O=gpurun_out/r02w11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/lib_3g8w.so GTC_WS_GROUPS=3 GTC_WS_DECW=8 GTC_WS_CTAS=1 >> $O/build.log 2>&1
GTC_LIB=/tmp/lib_3g8w.so timeout 300 python tools/loopback_bench.py --world 2 --steps 30 > $O/lb2.log 2>&1
GTC_LIB=/tmp/lib_3g8w.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_step_ws_group -s 20 -c 1 -o $O/ws_lb2 python tools/loopback_bench.py --world 2 --steps 30 > $O/ncu.log 2>&1
