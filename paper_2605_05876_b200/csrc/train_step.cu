// train_step.cu -- placeholder for the fused training-step kernels
