echo "fixed coords"; SSA_TC_DEBUG=1025 CUDA_LAUNCH_BLOCKING=1 timeout 60 python scripts/tc_debug.py 32 2>&1 | tail -1
echo "fixed coords noswz"; SSA_TC_BMODE=1 SSA_TC_DEBUG=1025 CUDA_LAUNCH_BLOCKING=1 timeout 60 python scripts/tc_debug.py 32 2>&1 | tail -1
