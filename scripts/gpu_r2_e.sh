bash scripts/ncu_box.sh xs512_m2 k_x_stream 1 1 env FM_XDIRECT=2 python scripts/prof_G.py 512 2
bash scripts/ncu_box.sh xs512_m4 k_x_stream 1 1 env FM_XDIRECT=4 python scripts/prof_G.py 512 2
