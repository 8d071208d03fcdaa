for pdl in 1 0 1 0; do echo "PDL=$pdl"; PNP_PDL=$pdl python scripts/cfg5_repeat.py 64; done
