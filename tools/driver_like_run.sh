# What the driver runs at round end, in one gpurun call: GPU suite, smoke, both bench arms (plain and under torchrun).
set -u
O=gpurun_out/driver_like
mkdir -p $O
( time timeout 1500 python -m pytest tests -x -q -m gpu ) > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 3 ) > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 3 ) > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?" >> $O/status
( time timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 ) > $O/bench_torchrun.jsonl 2> $O/bench_torchrun.err; echo "torchrun rc=$?" >> $O/status
cat $O/status; tail -3 $O/pytest_gpu.log; tail -4 $O/bench.err
