NSS_GP_DBG=4 python scripts/gp_kernel_probe.py 296
NSS_GP_DBG=4 python scripts/gp_kernel_probe.py 592
