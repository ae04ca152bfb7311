timeout 600 python tools/c4_order.py ablate C4
timeout 900 python tools/c4_order.py ablate C2
