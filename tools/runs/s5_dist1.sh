# the N > 1 bench path (NCCL init, barriers, max-over-ranks reductions) exercised with one rank under torchrun
for c in c4 c2 c3 c5; do
  FL1_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/s5_dist1_$c.json 2> gpurun_out/s5_dist1_$c.err; echo dist1_${c}_rc=$?; tail -c 300 gpurun_out/s5_dist1_$c.json; echo; tail -3 gpurun_out/s5_dist1_$c.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 --config c2 > gpurun_out/s5_dist1_ref.json 2> gpurun_out/s5_dist1_ref.err; echo ref_rc=$?; tail -c 200 gpurun_out/s5_dist1_ref.json
