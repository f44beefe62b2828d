for t in "TAG=packed" "RXG_CHUNK_SHAPE=5" "RXG_NO_PACKED=1"; do env $t TAG="$t" python tools/sweep_e.py; done
