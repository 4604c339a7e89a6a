echo "== default (early publish)"; timeout 120 python tools/parity_quick.py gs2d9p | tail -1; timeout 60 python tools/profile_run.py --config 4 --reps 2 | tail -1
echo "== nosleep"; TVSTENCIL_LIB=build/var/lib_nosleep.so timeout 120 python tools/parity_quick.py gs2d9p | tail -1; TVSTENCIL_LIB=build/var/lib_nosleep.so timeout 60 python tools/profile_run.py --config 4 --reps 2 | tail -1
