// Host<->device transfer options for the pageable-buffer sweep (development aid):
// pageable cudaMemcpy, cudaHostRegister cost + registered copies, pinned copies,
// and multi-threaded host memcpy into a pinned staging buffer.
// build: nvcc -O2 -o tools/h2d_probe tools/h2d_probe.cu -Xcompiler -pthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? std::atof(argv[1]) : 4.3) * 1e9;
    char* host = (char*)std::malloc(bytes);
    std::memset(host, 1, bytes);   // touch the pages
    char* dev = nullptr;
    cudaMalloc(&dev, bytes);
    cudaStream_t st;
    cudaStreamCreate(&st);
    double t0 = now();
    cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
    double t1 = now();
    std::printf("pageable H2D  %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
    t0 = now();
    cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost);
    t1 = now();
    std::printf("pageable D2H  %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
    t0 = now();
    cudaHostRegister(host, bytes, cudaHostRegisterDefault);
    t1 = now();
    std::printf("cudaHostRegister %.3f s (%.1f GB/s)\n", t1 - t0, bytes / (t1 - t0) / 1e9);
    t0 = now();
    cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    t1 = now();
    std::printf("registered H2D %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
    t0 = now();
    cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    t1 = now();
    std::printf("registered D2H %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
    t0 = now();
    cudaHostUnregister(host);
    t1 = now();
    std::printf("cudaHostUnregister %.3f s\n", t1 - t0);
    // multi-threaded host memcpy into a pinned buffer
    const size_t sb = 256u << 20;
    char* pin = nullptr;
    cudaMallocHost(&pin, sb);
    char* src2 = (char*)std::malloc(sb);
    std::memset(src2, 2, sb);
    for (int nt : {1, 2, 4, 8, 16, 32}) {
        t0 = now();
        for (int rep = 0; rep < 4; ++rep) {
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t)
                th.emplace_back([&, t] {
                    const size_t a = sb * t / nt, b = sb * (t + 1) / nt;
                    std::memcpy(pin + a, src2 + a, b - a);
                });
            for (auto& x : th) x.join();
        }
        t1 = now();
        std::printf("host memcpy -> pinned, %2d threads: %.1f GB/s\n", nt, 4.0 * sb / (t1 - t0) / 1e9);
    }
    std::printf("hardware threads %u\n", std::thread::hardware_concurrency());
    return 0;
}
