for c in cfg1 cfg3; do for v in "$@"; do CFG=$c ROPESLR_LIBRARY=_ab/$v.so timeout 300 python scripts/exp_k3ab.py 2>&1 | tail -2; done; done
