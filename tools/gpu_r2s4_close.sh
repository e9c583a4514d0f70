# session-4 closing set with the B = 48 x 3 headline: launch list of the default workload, ncu --set full of one
# B = 16 HMult + HRot step (summary), sanity of the N = 2 torchrun path (2 ranks sharing cuda:0, gloo)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4c_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -s 30 -c 30 -f -o /tmp/s4c_full \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/s4c_ncu_all.log 2>&1
python tools/ncu_summary.py /tmp/s4c_full.ncu-rep gpurun_out/s4c_ncu_all_kernels_summary.csv
CK32_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/s4c_torchrun2.json 2> gpurun_out/s4c_torchrun2.err
tail -c 400 gpurun_out/s4c_torchrun2.json
python tools/launch_table.py gpurun_out/s4c_launches_default.csv | head -14
