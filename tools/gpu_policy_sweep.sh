for f2c in 0.1225 0.16 0.2; do for c2f in 0.36 0.6 1.0 2.0; do
HSDE_POL_F2C=$f2c HSDE_POL_C2F=$c2f python tools/policy_sweep.py 2>&1 | tail -1
done; done
