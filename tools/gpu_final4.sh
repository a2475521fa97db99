#!/bin/bash
# final round-1 measurements on a 4-GPU box (tests, smoke, bench 1/2/4, reference arm, ER 2/4, ncu of the final kernel)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo "n1 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref_n1.json 2> gpurun_out/final/ref_n1.err; echo "ref rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/final/bench_n$N.json 2> gpurun_out/final/bench_n$N.err; echo "n$N rc=$?"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --no-alt-labeling --graph er --mode bfs --scale 28 --scaling strong --theta 64 --steps 16 > gpurun_out/final/er28_n2.json 2> gpurun_out/final/er28_n2.err; echo "er2 rc=$?"
for f in bench_n1 bench_n2 bench_n4 er28_n2; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/final/$f.json') if l.startswith('{')][0]); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d.get('cpu_baseline',{}).get('value'))"; done
cat gpurun_out/final/ref_n1.json
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-alt-labeling > gpurun_out/final/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-alt-labeling > gpurun_out/final/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/ncu_target.py 24 dobfs > gpurun_out/final/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o gpurun_out/prof_bfs_r01 -f python tools/ncu_target.py 24 dobfs > gpurun_out/final/ncu_full.log 2>&1; echo "full rc=$?"
