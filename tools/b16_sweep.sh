# INT8 B=16 activation-mode / plan experiments (A16 mask bits: 0 QKV, 1 attn-out, 2 up, 3 down)
bash tools/knob_sweep.sh "X=0 DSINF_A16_MASK=0xf DSINF_A16_MASK=0xf,DSINF_LN_STREAM=1 DSINF_A16_MASK=0xf,DSINF_STAGES_QKV=3 DSINF_PDL_MASK=0xaf" --dtype int8 --batch 16
bash tools/knob_sweep.sh "X=0 DSINF_LN_STREAM=1 DSINF_PDL_MASK=0xaf DSINF_STAGES_O=3" --dtype int8 --batch 8
bash tools/knob_sweep.sh "X=0 DSINF_PDL_MASK=0xaf DSINF_PDL_MASK=0x2d" --dtype fp16 --batch 16
