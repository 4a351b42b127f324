timeout 900 python tools/components.py c2 c3h c3 2>&1 | tail -2
