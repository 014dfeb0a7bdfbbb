TSQ_LIB=build_var/libtsq_phase.so TSQ_DEBUG_LEVELS=1 TSQ_HOST_LEVELS=1 python scripts/profile_sort.py uniform 67108864 2 2>&1 | tail -15
TSQ_LIB=build_var/libtsq_phase.so TSQ_DEBUG_LEVELS=1 TSQ_HOST_LEVELS=1 python scripts/profile_sort.py uniform 1048576 2 2>&1 | tail -8
