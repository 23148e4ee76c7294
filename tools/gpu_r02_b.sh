# round 2: C5 residual stability, default bench, warm ncu traffic captures (N=1 kernel, loopback fused kernel)
set -x
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
GTC_C5_REPORT=$O/c5.json timeout 1500 python -m pytest tests/test_gpu_c5.py -q -s > $O/c5.log 2>&1; echo "EXIT $?" >> $O/c5.log
timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 python bench.py --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > $O/plain_n1.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics $M -k regex:gtc_encode_tile_kernel -s 300 -c 30 \
  --csv --log-file $O/traffic_n1.csv python bench.py --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > $O/ncu_n1.log 2>&1
timeout 600 python tools/loopback_bench.py --world 2 --steps 60 > $O/lb2.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics $M -k regex:gtc_step_p2p_group -s 30 -c 20 \
  --csv --log-file $O/traffic_lb2.csv python tools/loopback_bench.py --world 2 --steps 60 > $O/ncu_lb2.log 2>&1
timeout 600 python tools/loopback_bench.py --world 4 --steps 60 > $O/lb4.log 2>&1
