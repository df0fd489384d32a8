for rep in 1 2; do for mb in 0 32 64 96; do echo "mb=$mb $(PO_L2PF_MB=$mb timeout 120 python tools/hit_once.py 2>&1 | tail -1)"; done; done
