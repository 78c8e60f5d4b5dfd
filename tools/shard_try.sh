#!/bin/bash
# usage: shard_try.sh NAME TILE [extra env...]
name=$1; tile=$2; shift 2
env MLAMR_TEST_VERBOSE=1 MLAMR_OVERLAP_REFRESH=0 MLAMR_L1_TILE=$tile "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29000 + RANDOM % 900)) tests/dist_gpu_worker.py $name 2>&1 | grep -E "differs|sharded == single|AssertionError" | sort | uniq -c | head -8
