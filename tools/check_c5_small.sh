# Functional check of bench.py --config c5 on a one-GPU box at reduced size: 1 rank, then
# 2 and 4 ranks on device 0 (peer transport over CUDA IPC between the processes).
set -x
mkdir -p gpurun_out/c5
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c5/smoke.txt 2>&1
PF_BENCH_C5_LEVELS=${LV:-7} timeout 600 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/c5/n1.txt 2>&1
for n in 2 4; do
PF_BENCH_DEVICE=0 PF_BENCH_C5_LEVELS=${LV:-7} timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 2 --warmup 3 > gpurun_out/c5/n$n.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph_cache or destroyed" > gpurun_out/c5/tests.txt 2>&1
