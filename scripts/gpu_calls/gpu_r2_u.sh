bash scripts/ncu_box2.sh xw512b k_x_warp 1 1 env FM_XDIRECT=7 python scripts/prof_G.py 512 2
