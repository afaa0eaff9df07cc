for i in 1 2; do for w in 2 4; do echo -n "W=$w: "; BSP_FILTER4=$w python tools/config_sweep.py C5 C2 --iters 20 2>/dev/null | grep -o "^C[0-9]*:\|[0-9.]* ms/iter" | tr '\n' ' '; echo; done; done
