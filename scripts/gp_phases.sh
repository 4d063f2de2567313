# phase clocks of the GP energy (measurement build, not the product library)
NSS_NVCC_EXTRA=-DNSS_GP_PHASES python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python scripts/gp_kernel_probe.py 296
python scripts/gp_kernel_probe.py 2960
