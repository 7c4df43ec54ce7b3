timeout 900 python tools/path_survey.py > gpurun_out/path_survey_r02.txt 2>&1; echo rc=$?; tail -30 gpurun_out/path_survey_r02.txt
