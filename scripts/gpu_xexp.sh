# persistent k_zf_fast with L2 prefetch of the next line group (K4 / compact J2 pass 1) against one CTA per group
for v in 0 1; do FM_ZF_PERSIST=$v python scripts/svk_check.py 256 k4; FM_ZF_PERSIST=$v python scripts/svk_check.py 512; done
for v in 0 1; do FM_ZF_PERSIST=$v CFG1_COMPACT=1 python scripts/cfg1_short.py 3 | tail -2; done
