P="timeout 120 python tools/power_probe.py"
$P jac3d27p 1024 1024 1024 --T 10 
$P jac3d27p 1024 1024 1024 --T 10 --fma allow
$P jac3d27p 160 160 160 --T 400 
$P jac3d27p 160 160 160 --T 400 --fma allow
$P jac3d27p 1024 1024 1024 --T 10 --algo naive
$P jac3d27p 1024 1024 1024 --T 10 --algo naive --fma allow
$P heat2d 16384 16384 --T 20 --algo naive
$P heat2d 16384 16384 --T 200
$P heat1d 268435456 --T 10 --algo naive
$P heat3d 1024 1024 1024 --T 10 --algo naive
$P jac2d9p 16384 16384 --T 20 --algo naive
