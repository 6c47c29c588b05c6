# A/B timing of multicolour-sweep builds (dev tool): bash scripts/ab_mc.sh [libs...]
libs="${@:-build/lib_*.so}"
for f in $libs; do echo "== $f"; OCMG_LIB=$PWD/$f timeout 120 python scripts/kbench.py --ops multicolour --iters 20; done
