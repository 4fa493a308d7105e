make -j8 >/dev/null 2>&1
ZINF_BENCH_SAME_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu --no-offload 2>&1 | grep -v Warning | grep "^{" | tail -1 > gpurun_out/bench_8rank_graph.json; echo rc $?; cut -c1-400 gpurun_out/bench_8rank_graph.json
