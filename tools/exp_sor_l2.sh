set -x
timeout 120 python tools/sor_time.py sor300 --kz 0
SOR3D_PERSIST=1 timeout 120 python tools/sor_time.py sor300 --kz 0
SOR3D_PERSIST=1 SOR3D_HINT=0 timeout 120 python tools/sor_time.py sor300 --kz 0
timeout 120 python tools/sor_time.py --shape 300,300,45 --kz 0
timeout 120 python tools/sor_time.py --shape 300,300,22 --kz 0
SOR3D_HINT=0 timeout 120 python tools/sor_time.py --shape 300,300,22 --kz 0
