# N > 1 bench paths on one GPU: ranks share the device over gloo (host-staged
# exchange; NCCL refuses two ranks on one GPU).  Strong and weak scaling,
# explicit and implicit, plus the reference arm under torchrun.
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$R --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --dist-backend gloo --cells 16x8x8 --steps 2 --warmup 3 --power-iters 20
$R --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --dist-backend gloo --cells 16x8x8 --steps 2 --warmup 3 --power-iters 20 --no-e2e
$R --nproc-per-node 2 --master-port 29513 bench.py --gpus 2 --dist-backend gloo --config c2 --cells 64x16 --scaling weak --steps 2 --warmup 3 --power-iters 20
$R --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 --dist-backend gloo --config c2 --cells 64x16 --integrator sdirk3 --steps 1 --warmup 1
$R --nproc-per-node 2 --master-port 29515 bench.py --gpus 2 --impl reference --config c1 --steps 1 --warmup 1
