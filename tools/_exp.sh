make -s >/dev/null 2>&1
for rep in 1 2 3; do for f in 1 2; do for sh in "14336 4096" "4096 14336"; do set -- $sh
GQSA_FEW=$f timeout 300 python tools/prof_layer.py --rows $1 --cols $2 --launches 1 --time 2>&1 | tail -1 | sed "s/^/FEW=$f /"; done; done; done
