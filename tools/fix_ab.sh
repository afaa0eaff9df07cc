# lambda-search placement A/B on C2: BSP_FIX_MODE 0 (k_hl_fix, full grid),
# 1 (in the fused kernel's last block), 2 (k_hl_fix on one block per SM)
for i in 1 2; do
  for m in 0 1 2; do
    echo -n "mode $m: bench-window "
    BSP_FIX_MODE=$m python tools/config_sweep.py C2 --iters 20 --warmup 5 2>/dev/null | grep -o "[0-9.]* ms/iter" | tr '\n' ' '
    echo -n " steady "
    BSP_FIX_MODE=$m python tools/config_sweep.py C2 --iters 2000 --warmup 100 2>/dev/null | grep -o "[0-9.]* ms/iter"
  done
done
