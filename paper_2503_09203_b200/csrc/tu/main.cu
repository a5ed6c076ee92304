// Translation unit main of libuuvb200.so (see UUV_TU in ../uuv_b200.cu).
#define UUV_TU 1
#include "../uuv_b200.cu"
