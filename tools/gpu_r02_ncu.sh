# round 2: ncu evidence on one GPU -- the N=1 launch list and full capture of the
# step kernel, and the ticketed N>1 kernel through a loopback group (world 2):
# warm DRAM traffic (20 back-to-back launches) and one full capture
set -x
O=${O:-gpurun_out/r02ncu2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B --steps 400 --warmup 5 > $O/plain_n1.jsonl 2> $O/plain_n1.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_n1.csv $B --steps 50 --warmup 5 > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_encode_tile_kernel -s 200 -c 1 -o $O/ncu_full_n1 $B --steps 300 --warmup 5 > $O/ncu_full_n1.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --cache-control none --clock-control none --metrics $M -k regex:gtc_encode_tile_kernel -s 300 -c 30 --csv --log-file $O/traffic_n1.csv $B --steps 400 --warmup 5 > $O/ncu_traffic_n1.log 2>&1
timeout 600 python tools/loopback_bench.py --world 2 --steps 60 > $O/lb2.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics $M -k regex:gtc_step_ticket_group -s 30 -c 20 --csv --log-file $O/traffic_lb2.csv python tools/loopback_bench.py --world 2 --steps 60 > $O/ncu_lb2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gtc_step_ticket_group -s 30 -c 1 -o $O/ncu_full_lb2 python tools/loopback_bench.py --world 2 --steps 40 > $O/ncu_full_lb2.log 2>&1
