TAG=${1:-p2}
set -x
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl.py -q -x --timeout=600 -p no:cacheprovider > gpurun_out/peer_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/peer_tests_$TAG.log
bash scripts/gpu_peer_bench.sh $TAG
