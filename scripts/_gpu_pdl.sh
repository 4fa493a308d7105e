# programmatic dependent launch: full GPU suite + smoke, then same-box A/B
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/_gpu_ab.sh ZI_PDL "0 1" 3
