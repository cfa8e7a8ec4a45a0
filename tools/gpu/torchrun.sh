# the driver's launch forms: torchrun with one rank (both arms) and the default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/tr_bench.json 2> gpurun_out/tr_bench.err; echo b=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/tr_ref.json 2> gpurun_out/tr_ref.err; echo r=$?
