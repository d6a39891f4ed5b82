# The round's ncu evidence on the final kernel: full captures of the
# headline, the L2-exceeding 16384-env batch and the floor instance, then
# the bench command's launch list (each after its command ran clean).
bash tools/ncu_capture.sh r2_render_step_humanoid_video_4096 Humanoid video 4096
bash tools/ncu_capture.sh r2_render_step_humanoid_video_16384 Humanoid video 16384
bash tools/ncu_capture.sh r2_render_step_ant_color_1024 Ant color 1024
bash tools/ncu_launches.sh
