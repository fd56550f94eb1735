for c in 1 2 4; do echo "ctas/SM $c"; PSD_SMALL_CTAS_PER_SM=$c PSD_LIB_VARIANT=debug timeout 120 python tools/small_stamps.py 2>&1 | grep stamps | head -2; done
