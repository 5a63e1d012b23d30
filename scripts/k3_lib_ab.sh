# A/B two library builds on K3 (ab_libs/lib_scalar.so vs ab_libs/lib_x2.so)
set -e
L=paper_1904_13342_b200/libtomograd_b200.so
cp ab_libs/lib_scalar.so $L; python scripts/k3_lib_ab.py save /tmp/k3_ref.pt scalar
cp ab_libs/lib_x2.so $L; python scripts/k3_lib_ab.py cmp /tmp/k3_ref.pt x2
cp ab_libs/lib_scalar.so $L; python scripts/k3_lib_ab.py cmp /tmp/k3_ref.pt scalar
cp ab_libs/lib_x2.so $L; python scripts/k3_lib_ab.py cmp /tmp/k3_ref.pt x2
