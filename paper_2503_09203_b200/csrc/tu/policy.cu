// Translation unit policy of libuuvb200.so (see UUV_TU in ../uuv_b200.cu).
#define UUV_TU 4
#include "../uuv_b200.cu"
