# round-2 closing measurement set (current defaults): full bench line, launch lists,
# ncu --set full summary of one B=16 HMult+HRot step, and the N=2 torchrun path (2 ranks sharing cuda:0, gloo)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default_final.json 2> gpurun_out/bench_default_final.err
tail -c 400 gpurun_out/bench_default_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b16_final.csv python bench.py --steps 2 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -s 30 -c 30 -f -o /tmp/final_full \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_all_final.log 2>&1
python tools/ncu_summary.py /tmp/final_full.ncu-rep gpurun_out/ncu_all_kernels_summary_final.csv
CK32_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/bench_torchrun2_gloo.json 2> gpurun_out/bench_torchrun2_gloo.err
tail -c 300 gpurun_out/bench_torchrun2_gloo.json
ls -la gpurun_out
