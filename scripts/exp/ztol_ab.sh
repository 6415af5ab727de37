for c in 131072 4194304; do
  APC_ZTOL_CHUNK=$c APC_SETUP_PROF=1 timeout 300 python scripts/prof_cfg.py 5 5 3 2>&1 | grep -o "aplicur_solve setup.*augment [0-9.]*\|setup_ms [0-9.]*" | sed "s/^/chunk=$c /"
done
