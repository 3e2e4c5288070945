bash tools/knob_sweep.sh "X=0 DSINF_STAGES_UP=4 DSINF_STAGES_UP=5 DSINF_STAGES_UP=6 DSINF_STAGES_UP=4,DSINF_STAGES_O=4 DSINF_STAGES_UP=4,DSINF_STAGES_DOWN=2 DSINF_STAGES_UP=4,DSINF_STAGES_QKV=3" --dtype int8
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_UP=4 DSINF_STAGES_UP=2" --dtype int8 --batch 2
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_UP=2 DSINF_STAGES_UP=3 DSINF_STAGES_QKV=3" --dtype int8 --batch 8
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_QKV=3 DSINF_STAGES_QKV=2 DSINF_STAGES_QKV=3,DSINF_STAGES_UP=2 DSINF_STAGES_QKV=3,DSINF_STAGES_O=6" --dtype fp16
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_QKV=3 DSINF_STAGES_UP=2 DSINF_STAGES_QKV=3,DSINF_STAGES_UP=2" --dtype fp16 --batch 8
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_UP=2 DSINF_STAGES_UP=2,DSINF_STAGES_QKV=3" --dtype fp16 --batch 16
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_QKV=3 DSINF_STAGES_UP=2" --config gpt2-1.5b --dtype fp16
bash tools/knob_sweep.sh "X=0 DSINF_STAGES_UP=4 DSINF_STAGES_UP=2" --config gpt2-1.5b --dtype int8
