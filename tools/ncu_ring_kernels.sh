# ncu --set full of the K3 kernels with an L2-resident batch (16 components at
# n = 20 = 32 MiB, no cache flush between replays): what bounds them when HBM does not
export SBW_K3_RING=0 SBW_PASSB_TC_MIN_N=17 SBW_K3_BATCH=16
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_passb_tc --launch-skip 6 -c 1 -o gpurun_out/ncu_passb_tc_l2 -f python tools/k3_probe.py 20x20 512 > gpurun_out/ncu_pb.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_tc_hybrid --launch-skip 6 -c 1 -o gpurun_out/ncu_passa_l2 -f python tools/k3_probe.py 20x20 512 > gpurun_out/ncu_pa.log 2>&1
ls -la gpurun_out
