for pr in 0 1; do echo "== priority $pr"; MOSHPIT_DIAG_AUX_PRIORITY=$pr timeout 600 python profiles/diag_probe.py 2>&1 | tail -1 | cut -c1-120; done
for pr in 0 1; do echo "== priority $pr"; MOSHPIT_DIAG_AUX_PRIORITY=$pr timeout 600 python profiles/diag_probe.py 2>&1 | tail -1 | cut -c1-120; done
