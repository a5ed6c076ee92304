// Translation unit serve of libuuvb200.so (see UUV_TU in ../uuv_b200.cu).
#define UUV_TU 5
#include "../uuv_b200.cu"
