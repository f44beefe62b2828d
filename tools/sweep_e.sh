for t in "RXG_NO_PACKED=1" "RXG_NO_PACKED=1 RXG_CHUNK_SHAPE=5" "RXG_NO_PACKED=1 RXG_CHUNK_SHAPE=8" "TAG=packed" "RXG_CHUNK_SHAPE=8"; do env $t TAG="$t" python tools/sweep_e.py; done
