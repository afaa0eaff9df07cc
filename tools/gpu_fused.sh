for k in 0 1 2 4 8 16 32 63; do echo "skip $k"; BSP_FUSED_SKIP=$k timeout 300 python tools/config_sweep.py C2 --iters 200 2>&1 | grep -v "^{" | grep -o "[0-9.]* ms/iter"; done
