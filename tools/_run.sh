timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file /tmp/st.csv python tools/sinr_time.py C2 20 > /dev/null 2>&1
python tools/ncu_summary.py launches /tmp/st.csv | head -12
