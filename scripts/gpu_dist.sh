# exercise the torchrun code paths of bench.py on the one available GPU
mkdir -p gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/dist_c2.json 2> gpurun_out/dist_c2.err; echo rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/dist_ref.json 2> gpurun_out/dist_ref.err; echo rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 1 --config c5 --steps 3 --warmup 3 > gpurun_out/dist_c5.json 2> gpurun_out/dist_c5.err; echo rc=$?
cut -c1-300 gpurun_out/dist_c2.json gpurun_out/dist_ref.json gpurun_out/dist_c5.json; tail -3 gpurun_out/dist_c2.err
