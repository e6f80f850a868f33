for r in 1 2; do
python scripts/time_scoresel.py 200
BSA_SCORESEL_DEBUG=1 python scripts/time_scoresel.py 200
BSA_LIB_VARIANT=s_rpt4 python scripts/time_scoresel.py 200
done
