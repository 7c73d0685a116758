python tools/step_time.py --scheme CS_E2LSH
python tools/step_time.py --scheme CS_E2LSH --keep 0
python tools/step_time.py --scheme CS_SRP
python tools/step_time.py --scheme CS_E2LSH --query
