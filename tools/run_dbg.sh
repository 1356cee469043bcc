for d in 0 1 8 9; do echo "== dbg $d"; ADAMAS_DBG=$d timeout 200 python tools/phase_profile.py --cluster 4 --layers 4 2>&1 ; done
