# the torchrun (distributed) path of bench.py on one GPU: gpurun -- "bash tools/gpu_dist1.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-companion > gpurun_out/$T/b2.json 2> gpurun_out/$T/b2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --config 4 --recordings 64 --blocks 100 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/b4.json 2> gpurun_out/$T/b4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --impl reference --steps 3 --warmup 3 > gpurun_out/$T/r2.json 2> gpurun_out/$T/r2.err
