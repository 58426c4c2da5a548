timeout 900 python tools/dbg_benchpath.py > gpurun_out/dbg_new.txt 2>&1
PKG_ROOT=$PWD/_old MODES=1 timeout 900 python tools/dbg_benchpath.py > gpurun_out/dbg_old.txt 2>&1
cat gpurun_out/dbg_new.txt gpurun_out/dbg_old.txt | grep -v Warn
