cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c34_build.log 2>&1
NSS_WPC=4 timeout 300 python scripts/wpc4_debug.py > gpurun_out/c34_debug.txt 2>&1
NSS_WPC=4 timeout 300 compute-sanitizer --tool memcheck python scripts/wpc4_debug.py > gpurun_out/c34_memcheck.txt 2>&1
