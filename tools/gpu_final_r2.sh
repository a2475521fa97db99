#!/bin/bash
# Round-2 closing measurements on a 4-GPU box: GPU test suite (device groups at
# p = 2/4), bench at N = 1/2/4 with the configs[2]/configs[3] series and the
# reference arm beside each, single-process device-group runs, ER (configs[4]).
cd $GRAFT_REPO_ROOT; O=gpurun_out/final_r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader | head -4 > $O/gpus.txt; nproc >> $O/gpus.txt; free -g | head -2 >> $O/gpus.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench1 rc=$?"
timeout 600 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref1 rc=$?"
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > $O/bench_n$N.json 2> $O/bench_n$N.err; echo "bench$N rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --impl reference > $O/ref_n$N.json 2> $O/ref_n$N.err; echo "ref$N rc=$?"
done
for P in 2 4; do timeout 900 python tools/group_bench.py $P $((24 + P / 2)) dobfs scramble 2>&1 | grep -v NCCL > $O/group_p$P.txt; DBFS_NVLS=1 timeout 900 python tools/group_bench.py $P $((24 + P / 2)) dobfs scramble 2>&1 | grep -v NCCL >> $O/group_p$P.txt; done
for N in 2 4; do timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --graph er --scale 28 --scaling strong --theta 64 --mode bfs --no-series --no-cpu-baseline --steps 2 > $O/bench_er_s28_bfs_n$N.json 2> $O/bench_er_n$N.err; echo "er$N rc=$?"; done
ls $O
