timeout 600 python tools/dbg_epoch.py 2>&1 | grep -v Warn > gpurun_out/dbg_epoch_new.txt
PKG_ROOT=$PWD/_old timeout 600 python tools/dbg_epoch.py 2>&1 | grep -v Warn > gpurun_out/dbg_epoch_old.txt
paste -d'\n' gpurun_out/dbg_epoch_new.txt gpurun_out/dbg_epoch_old.txt | head -80
