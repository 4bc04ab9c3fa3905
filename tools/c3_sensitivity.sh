#!/bin/bash
# C3 trajectory sensitivity to the compressed views' precision (CPU, the
# unmodified reference via oracle/_ref/golden_big): fp32-rounded projectors
# and views, and a 1e-6 relative perturbation of them.  Compare rec_err.f64
# against tests/golden/c3_full.npz (tools/c3_sensitivity.py).
B=oracle/_ref/golden_big
ARGS="100000 20000 50 0 1 0.01 1 50 70 2 100 5 1 4"
GOLDEN_VIEWS_F32=1 $B /tmp/sens_f32 $ARGS > /tmp/sens_f32/log 2>&1 &
GOLDEN_VIEWS_PERTURB=1e-6 $B /tmp/sens_p1e6 $ARGS > /tmp/sens_p1e6/log 2>&1 &
wait
# Range-finder perturbation (multithreaded fp64 contractions, views exact):
ARGS30="100000 20000 50 0 1 0.01 1 50 70 2 30 5 1 4"
GOLDEN_RF_PERTURB=1e-6 $B /tmp/rf_1e6 $ARGS30 > /tmp/rf_1e6/log 2>&1 &
GOLDEN_RF_PERTURB=1e-7 $B /tmp/rf_1e7 $ARGS30 > /tmp/rf_1e7/log 2>&1 &
wait
