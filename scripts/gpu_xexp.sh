# compact-J2 pass 1 register budget: 2 / 3 / 4 CTAs per SM (lib_exp builds; measured 1.31 / 1.31 / 1.66 ms at 256^3, 3 kept)
for mb in 3 4 2; do cp paper_1603_08893_b200/lib_exp/j2c$mb.so paper_1603_08893_b200/lib/libfftmech_b200.so
  echo "j2c minb=$mb"; python scripts/svk_check.py 256 j2c; python scripts/svk_check.py 512 j2c; done
