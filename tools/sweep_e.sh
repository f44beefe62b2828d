# (e) device time vs size: packed layout (default) against the row layout, same box
for t in "TAG=packed" "RXG_NO_PACKED=1"; do env $t TAG="$t" python tools/sweep_e.py; done
