bash scripts/ncu_box.sh xw512 k_x_warp 1 1 env FM_XDIRECT=7 python scripts/prof_G.py 512 2
