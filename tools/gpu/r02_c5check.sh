cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
   bench.py --gpus 1 --config c5 --c5-log2 27 --steps 3 --warmup 2 > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err
echo "c5 torchrun rc=$?"; tail -3 gpurun_out/c5_n1.err
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/gpus2.json 2> gpurun_out/gpus2.err
echo "gpus2 rc=$?"; cat gpurun_out/gpus2.json; tail -2 gpurun_out/gpus2.err
timeout 300 python bench.py --impl reference --config c5 --steps 2 --warmup 1 > gpurun_out/c5_ref.json 2>&1
echo "c5 ref rc=$?"
