timeout 600 python tools/ab_host_slots.py
timeout 300 python tools/e2e_bound.py
