run() { echo "== $*"; env "$@" timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/p2p_bw.py 2>&1 | grep "nccl send"; }
run X=1
run NCCL_MIN_P2P_NCHANNELS=16
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 NCCL_NCHANNELS_PER_PEER=32
run NCCL_P2P_NVL_CHUNKSIZE=2097152
run NCCL_BUFFSIZE=33554432 NCCL_MIN_P2P_NCHANNELS=16
run NCCL_P2P_USE_CUDA_MEMCPY=1
run NCCL_PROTO=Simple NCCL_MIN_P2P_NCHANNELS=16
