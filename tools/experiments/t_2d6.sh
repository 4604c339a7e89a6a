timeout 120 python tools/parity_quick.py heat2d | tail -1
echo "== seg256"; for d in 4 5 6 7 8; do timeout 60 python tools/profile_run.py --config 3 --depth $d --reps 3 | tail -1; done
for sg in 512 128; do echo "== seg$sg"; TVSTENCIL_LIB=build/var/lib_s$sg.so timeout 120 python tools/parity_quick.py heat2d | tail -1; for d in 6 8; do TVSTENCIL_LIB=build/var/lib_s$sg.so timeout 60 python tools/profile_run.py --config 3 --depth $d --reps 3 | tail -1; done; done
