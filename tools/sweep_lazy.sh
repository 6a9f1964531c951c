# lazy-QR threshold slack (kappa; no bit of the result depends on it) and the ring kernel, C4 / C5
for kap in 4 8 12; do echo "kappa=$kap: $(RID_QRCP_LAZY=1 RID_QRCP_KAPPA=$kap python tools/qr_time.py C4 C5 2>&1 | awk "{print \$6}" | tr '\n' ' ')"; done
echo "ring: $(RID_QRCP_LAZY=0 python tools/qr_time.py C4 C5 2>&1 | awk "{print \$6}" | tr '\n' ' ')"
