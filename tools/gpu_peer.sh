#!/bin/bash
# peer-engine check at N GPUs: oracle parity of host vs peer engines, then the bench line
N=${1:-2}; S=${2:-18}; BS=${3:-24}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py $S > gpurun_out/peer_check_n$N.log 2>&1; echo "check rc=$?"; grep -E "root|DIST|built|disagree|Error|error" gpurun_out/peer_check_n$N.log | head -60
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $N --scale $BS --steps 16 --warmup 3 > gpurun_out/bench_peer_n$N.json 2> gpurun_out/bench_peer_n$N.err; echo "bench rc=$?"; cat gpurun_out/bench_peer_n$N.json; tail -5 gpurun_out/bench_peer_n$N.err
